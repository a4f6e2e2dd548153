# column-chunked tensor-core screen: guarded first runs
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "c1_free_running and tensor_chunked" > gpurun_out/gtest43a.log 2>&1; echo "c1 rc=$?"; tail -3 gpurun_out/gtest43a.log
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "tensor_chunked" > gpurun_out/gtest43.log 2>&1; echo "all rc=$?"; tail -3 gpurun_out/gtest43.log
for C in c5 c4 c3; do timeout 300 python bench.py --config $C --engine tensor_chunked --no-cpu-baseline --no-e2e --stats-out gpurun_out/st43_$C.json > gpurun_out/b43_$C.json 2> gpurun_out/b43_$C.err; python -c "
import json; j=json.load(open('gpurun_out/b43_$C.json')); print('$C tcc', round(j['value'],2), round(j['ms_per_step'],3), round(j['roofline']['avg_launch_ms'],3))" || tail -3 gpurun_out/b43_$C.err; done
