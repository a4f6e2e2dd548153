# quick bench: tests + configs given as args
T=$1; shift
if [ "$T" = "t" ]; then timeout 400 python -m pytest tests -m gpu -x -q > gpurun_out/tq.log 2>&1; tail -1 gpurun_out/tq.log; fi
for C in "$@"; do timeout 600 python bench.py --config $C --no-cpu-baseline --no-e2e > gpurun_out/bq_$C.json 2> gpurun_out/bq_$C.err; python -c "
import json; j=json.load(open('gpurun_out/bq_$C.json')); print('$C', round(j['value'],2), round(j['ms_per_step'],3), round(j['roofline']['avg_launch_ms'],3), round(j['roofline']['frac'],4))" || tail -3 gpurun_out/bq_$C.err; done
