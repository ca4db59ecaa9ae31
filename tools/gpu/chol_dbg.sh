cd $GRAFT_REPO_ROOT
HS_GEMM_PERSIST=1 timeout 300 python tools/gpu/chol_det.py
for k in 1 2; do for v in 1 0; do
echo "== HS_GEMM_PERSIST=$v"; HS_GEMM_PERSIST=$v timeout 300 python tools/chol_bench.py --n 32768 --b 512 --slices 0 --reps 2 2>&1 | grep -v "^chol " ; done; done
timeout 1200 python -m pytest tests -m gpu -q -k "chol or factor or spd or potf or gemm or substitution or not_spd or singular or finite or oz or cyclic or group or fullsize" 2>&1 | grep -E "FAILED|passed|failed|Error|assert" | head -40
HS_CHOL_TIMING=1 timeout 300 python tools/chol_bench.py --n 32768 --b 512 --slices 0 --reps 1 > gpurun_out/chol_timing.txt 2>&1
