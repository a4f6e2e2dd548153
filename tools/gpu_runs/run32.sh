# screen engine: parity on the engine-parametrised tests, then C3/C4/C5 benches (walk vs screen)
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "screen" > gpurun_out/gtest32.log 2>&1; tail -15 gpurun_out/gtest32.log
for C in c3 c4 c5; do for E in screen; do
timeout 600 python bench.py --config $C --engine $E --no-cpu-baseline --no-e2e --stats-out gpurun_out/st32_${C}_$E.json > gpurun_out/b32_${C}_$E.json 2> gpurun_out/b32_${C}_$E.err; python -c "
import json; j=json.load(open('gpurun_out/b32_${C}_$E.json')); print('$C $E', round(j['value'],2), round(j['ms_per_step'],3), round(j['roofline']['avg_launch_ms'],3), round(j['roofline']['frac'],4))" || tail -5 gpurun_out/b32_${C}_$E.err; done; done
