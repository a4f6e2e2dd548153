CMD="python bench.py --config c3 --engine tensor_screen --steps 9 --warmup 3 --no-e2e --no-cpu-baseline"
for K in k_mti_tc k_resolve; do
ncu --set full --clock-control none --import-source on -k regex:"$K" -s 8 -c 1 -o /tmp/prof_$K $CMD > gpurun_out/ncu36_$K.log 2>&1
ncu -i /tmp/prof_$K.ncu-rep --page raw --csv > gpurun_out/raw36_$K.csv 2>/dev/null
ncu -i /tmp/prof_$K.ncu-rep --page source --print-source cuda,sass --csv 2>/dev/null | gzip > gpurun_out/src36_$K.csv.gz
done
