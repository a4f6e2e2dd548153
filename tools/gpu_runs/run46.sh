timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "c1_free_running and tensor_chunked" > gpurun_out/gtest46a.log 2>&1; echo "c1 rc=$?"; tail -2 gpurun_out/gtest46a.log
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "tensor_chunked" > gpurun_out/gtest46.log 2>&1; echo "rc=$?"; tail -2 gpurun_out/gtest46.log
for C in c5 c4 c3; do timeout 300 python bench.py --config $C --engine tensor_chunked --no-cpu-baseline --no-e2e --stats-out gpurun_out/st46_$C.json > gpurun_out/b46_$C.json 2> gpurun_out/b46_$C.err; python -c "
import json; j=json.load(open('gpurun_out/b46_$C.json')); print('$C tcc', round(j['value'],2), round(j['ms_per_step'],3), round(j['roofline']['avg_launch_ms'],3))" || tail -3 gpurun_out/b46_$C.err; done
CMD="python bench.py --config c5 --engine tensor_chunked --steps 4 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_tcc" -s 4 -c 1 -o /tmp/prof46 $CMD > gpurun_out/ncu46.log 2>&1
ncu -i /tmp/prof46.ncu-rep --page raw --csv > gpurun_out/raw46_k_tcc.csv 2>/dev/null
ncu -i /tmp/prof46.ncu-rep --page source --print-source cuda,sass --csv 2>/dev/null | gzip > gpurun_out/src46_k_tcc.csv.gz
