# round 2 re-entry: tcc parity subset + bench of walk vs tcc on C3/C4/C5
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "tensor_chunked" > gpurun_out/gtest47.log 2>&1; echo "tcc tests rc=$?"; tail -2 gpurun_out/gtest47.log
for C in c5 c4 c3; do for E in tensor_chunked auto; do timeout 400 python bench.py --config $C --engine $E --no-cpu-baseline --no-e2e --stats-out gpurun_out/st47_${C}_$E.json > gpurun_out/b47_${C}_$E.json 2> gpurun_out/b47_${C}_$E.err; python -c "
import json; j=json.load(open('gpurun_out/b47_${C}_$E.json')); print('$C $E', round(j['value'],2), round(j['ms_per_step'],3), round(j['roofline']['avg_launch_ms'],3))" || tail -3 gpurun_out/b47_${C}_$E.err; done; done
