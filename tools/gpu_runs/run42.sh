# dense pass with R rows per lane (iteration 1 and knori-)
timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q -k "not screen and not tensor" > gpurun_out/gtest42.log 2>&1; tail -2 gpurun_out/gtest42.log
timeout 600 python bench.py > gpurun_out/bench42.json 2> gpurun_out/bench42.err; python -c "
import json; j=json.load(open('gpurun_out/bench42.json')); print(j['value'], j['ms_per_step'], j['roofline']['avg_launch_ms'], j['e2e']['value'], j['e2e']['phases'])" || tail -3 gpurun_out/bench42.err
for C in c3 c4; do timeout 600 python bench.py --config $C --prune none --no-cpu-baseline --no-e2e > gpurun_out/b42_${C}_none.json 2>&1; python -c "
import json; j=json.load(open('gpurun_out/b42_${C}_none.json')); print('$C none', round(j['value'],2), round(j['ms_per_step'],3), round(j['roofline']['avg_launch_ms'],3), round(j['roofline']['frac'],4))"; done
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches42.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
