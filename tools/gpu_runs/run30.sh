# round-2 re-entry check: full GPU suite, default bench, quick C4/C5 benches
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 2400 python -m pytest tests -m gpu -x -q --durations=15 > gpurun_out/gtest30.log 2>&1; tail -25 gpurun_out/gtest30.log
timeout 600 python bench.py > gpurun_out/bench30.json 2> gpurun_out/bench30.err; tail -c 1500 gpurun_out/bench30.json; tail -3 gpurun_out/bench30.err
bash tools/qb.sh n c4 c5
