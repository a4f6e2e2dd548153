# closing check of the committed build: smoke(), the d = 32 and strict-parity subsets, the default bench line
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 500 python -m pytest tests/test_gpu_parity.py -x -q -k "table_head or B1 or B2 or c1_free or c2_free or (spectral and cuda) or two_gpus or graph or nccl" > gpurun_out/gtest65.log 2>&1; echo "subset rc=$?"; tail -1 gpurun_out/gtest65.log
python bench.py > gpurun_out/bench65_c3.json 2> gpurun_out/bench65_c3.err; echo "bench rc=$?"
python -c "
import json; j=json.load(open('gpurun_out/bench65_c3.json')); print(round(j['value'],1), round(j['roofline']['avg_launch_ms'],3), round(j['roofline']['frac'],4), 'e2e', round(j['e2e']['value'],1), j['roofline']['traffic'])"
