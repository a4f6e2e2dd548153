# ncu of the exception-path walk on C3 with a re-sort after every pass (exceptions = movers)
bash tools/ncu_capture.sh c3 r2e "k_walk" 8 --resort-fraction 0.01
