# old walk + swizzled DP=8 staging, batched flush loads, deferred claims, ldg256, cmax prefetch
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "c1_free or c2_free or spectral or c5_shaped or B1 or B2 or B5 or dims or ragged or k1 or resum or resort or graph" > gpurun_out/gtest24.log 2>&1; tail -1 gpurun_out/gtest24.log
for C in c3 c4 c5; do timeout 600 python bench.py --config $C --no-cpu-baseline --no-e2e --stats-out gpurun_out/st24_${C}.json > gpurun_out/b24_${C}.json 2> gpurun_out/b24_${C}.err; python -c "
import json; j=json.load(open('gpurun_out/b24_${C}.json')); print('$C', round(j['value'],2), round(j['ms_per_step'],3), round(j['roofline']['avg_launch_ms'],3), round(j['roofline']['frac'],4))" || tail -3 gpurun_out/b24_${C}.err; done
