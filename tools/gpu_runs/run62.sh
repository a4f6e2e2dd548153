# final call of round 2: whole GPU suite, the bench lines of C3 (default command) / C4 / C5, the ncu
# launch list of the default bench command, one --set full capture of C3's and C4's walk
python -m pytest tests -m gpu -x -q > gpurun_out/gputest_final.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/gputest_final.log
python bench.py > gpurun_out/bench_final_c3.json 2> gpurun_out/bench_final_c3.err; echo "bench c3 rc=$?"
python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/bench_final_c3_reference.json 2> gpurun_out/bench_final_c3_reference.err; echo "reference rc=$?"
for C in c4 c5; do
  timeout 900 python bench.py --config $C --no-cpu-baseline --stats-out gpurun_out/stats_final_$C.json > gpurun_out/bench_final_$C.json 2> gpurun_out/bench_final_$C.err; echo "bench $C rc=$?"
done
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_final_c3.csv python bench.py --no-cpu-baseline > gpurun_out/ncu_launch_c3.log 2>&1; echo "launch list rc=$?"
timeout 600 bash tools/ncu_capture.sh c3 final k_walk 8
timeout 900 bash tools/ncu_capture.sh c4 final k_walk 8
for f in gpurun_out/bench_final_*.json; do python - "$f" <<'PY'
import json,sys
j=json.load(open(sys.argv[1])); r=j.get('roofline',{}); e=j.get('e2e',{})
print(sys.argv[1], round(j.get('value',0),2), j.get('unit'), 'pass', round(r.get('avg_launch_ms',0),3), r.get('kernel'), 'frac', round(r.get('frac',0),4), 'e2e', e.get('value'))
PY
done
