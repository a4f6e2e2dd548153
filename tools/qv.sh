# A/B variants: tools/qv.sh "base t640 t1024" "c3 c4"  (base = the in-tree build)
for V in $1; do
  if [ "$V" = base ]; then L=""; else L="$PWD/variants/$V.so"; fi
  for C in $2; do
    KM_LIB=$L timeout 600 python bench.py --config $C --no-cpu-baseline --no-e2e > gpurun_out/bv_${V}_$C.json 2> gpurun_out/bv_${V}_$C.err
    python -c "
import json; j=json.load(open('gpurun_out/bv_${V}_$C.json')); print('$V $C', round(j['value'],2), round(j['ms_per_step'],3), round(j['roofline']['avg_launch_ms'],3), round(j['roofline']['frac'],4))" || tail -2 gpurun_out/bv_${V}_$C.err
  done
done
