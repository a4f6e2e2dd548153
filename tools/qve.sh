# A/B variants with extra bench args: tools/qve.sh "base v1 v2" "c3 c4" "--engine screen"
for V in $1; do
  if [ "$V" = base ]; then L=""; else L="$PWD/variants/$V.so"; fi
  for C in $2; do
    KM_LIB=$L timeout 600 python bench.py --config $C --no-cpu-baseline --no-e2e $3 --stats-out gpurun_out/sv_${V}_$C.json > gpurun_out/bv_${V}_$C.json 2> gpurun_out/bv_${V}_$C.err
    python -c "
import json; j=json.load(open('gpurun_out/bv_${V}_$C.json')); print('$V $C', round(j['value'],2), round(j['ms_per_step'],3), round(j['roofline']['avg_launch_ms'],3), round(j['roofline']['frac'],4))" || tail -2 gpurun_out/bv_${V}_$C.err
  done
done
