# exact-order sums via per-block stable lists; iteration-1 sums before the first re-bucketing
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_ti.py -x -q -k "not screen" > gpurun_out/gtest38.log 2>&1; tail -3 gpurun_out/gtest38.log
timeout 600 python bench.py > gpurun_out/bench38.json 2> gpurun_out/bench38.err; python -c "
import json; j=json.load(open('gpurun_out/bench38.json')); print(j['value'], j['ms_per_step'], j['roofline']['avg_launch_ms'], j['e2e']['value'], j['e2e']['phases'])" || tail -3 gpurun_out/bench38.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches38.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
timeout 1800 python -m pytest tests/test_gpu_fullsize.py -x -q -k "cuda" > gpurun_out/gfull38.log 2>&1; tail -3 gpurun_out/gfull38.log
