set -x
nproc; nvidia-smi --query-gpu=name,clocks.sm --format=csv
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -2 gpurun_out/smoke.log
timeout 1200 python -m pytest tests -m gpu -x -q --deselect "tests/test_gpu_fullsize.py::test_full_size_trajectory[c4]" --deselect "tests/test_gpu_fullsize.py::test_full_size_trajectory[c5]" --durations=15 > gpurun_out/gtest.log 2>&1; tail -25 gpurun_out/gtest.log
python bench.py --steps 20 --warmup 5 > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err; tail -c 1500 gpurun_out/bench_c3.json; tail -5 gpurun_out/bench_c3.err
python bench.py --prune none --no-cpu-baseline --no-e2e > gpurun_out/bench_c3_none.json 2>&1
python bench.py --config c4 --prune none --no-cpu-baseline --no-e2e > gpurun_out/bench_c4_none.json 2>&1
python bench.py --config c4 --no-cpu-baseline --no-e2e > gpurun_out/bench_c4.json 2>&1
/usr/bin/time -v python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/ref_c3.json 2> gpurun_out/ref_c3.err; tail -c 800 gpurun_out/ref_c3.json; grep -E "Elapsed|Maximum resident" gpurun_out/ref_c3.err
