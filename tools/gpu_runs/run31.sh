# fresh ncu --set full + source page of the C3 walk (re-entry baseline)
bash tools/ncu_capture.sh c3 r2d "k_walk" 8
