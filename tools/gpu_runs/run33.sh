# screen engine C3: launch list + full captures of k_screen and k_resolve (source pages)
CMD="python bench.py --config c3 --engine screen --steps 9 --warmup 3 --no-e2e --no-cpu-baseline"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c3_scr.csv $CMD > /dev/null 2>&1
for K in k_screen k_resolve; do
ncu --set full --clock-control none --import-source on -k regex:"$K" -s 8 -c 1 -o /tmp/prof_$K $CMD > gpurun_out/ncu_$K.log 2>&1
ncu -i /tmp/prof_$K.ncu-rep --page raw --csv > gpurun_out/raw_c3_$K.csv 2>/dev/null
ncu -i /tmp/prof_$K.ncu-rep --page source --print-source cuda,sass --csv 2>/dev/null | gzip > gpurun_out/src_c3_$K.csv.gz
done
