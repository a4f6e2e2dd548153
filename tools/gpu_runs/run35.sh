# tensor-screen engine: parity on the engine-parametrised tests, then C3/C4 benches + launch list
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "tensor_screen" > gpurun_out/gtest35.log 2>&1; tail -15 gpurun_out/gtest35.log
for C in c3 c4; do for E in tensor_screen; do
timeout 600 python bench.py --config $C --engine $E --no-cpu-baseline --no-e2e --stats-out gpurun_out/st35_${C}_$E.json > gpurun_out/b35_${C}_$E.json 2> gpurun_out/b35_${C}_$E.err; python -c "
import json; j=json.load(open('gpurun_out/b35_${C}_$E.json')); print('$C $E', round(j['value'],2), round(j['ms_per_step'],3), round(j['roofline']['avg_launch_ms'],3), round(j['roofline']['frac'],4))" || tail -5 gpurun_out/b35_${C}_$E.err; done; done
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c3_tcs.csv python bench.py --config c3 --engine tensor_screen --steps 9 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
