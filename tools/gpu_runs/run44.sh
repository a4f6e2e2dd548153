timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "tensor_chunked" > gpurun_out/gtest44.log 2>&1; echo "rc=$?"; tail -3 gpurun_out/gtest44.log
CMD="python bench.py --config c5 --engine tensor_chunked --steps 4 --warmup 3 --no-e2e --no-cpu-baseline"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches44_c5.csv $CMD > /dev/null 2>&1
for K in k_tcc k_resolve; do
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$K" -s 4 -c 1 -o /tmp/prof44_$K $CMD > gpurun_out/ncu44_$K.log 2>&1
ncu -i /tmp/prof44_$K.ncu-rep --page raw --csv > gpurun_out/raw44_$K.csv 2>/dev/null
ncu -i /tmp/prof44_$K.ncu-rep --page source --print-source cuda,sass --csv 2>/dev/null | gzip > gpurun_out/src44_$K.csv.gz
done
