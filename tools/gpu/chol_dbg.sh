cd $GRAFT_REPO_ROOT
timeout 300 python tools/diag_timing.py > gpurun_out/diag_timing.txt 2>&1
timeout 300 python tools/gpu/chol_det.py
for k in 1 2; do timeout 300 python tools/chol_bench.py --n 32768 --b 512 --slices 0 8 --reps 2 2>&1 | grep -v "^chol " ; done
timeout 1200 python -m pytest tests -m gpu -q -k "chol or factor or spd or potf or gemm or substitution or not_spd or singular or finite or oz or cyclic or group or fullsize or diag" 2>&1 | grep -E "FAILED|passed|failed|Error|assert" | head -20
