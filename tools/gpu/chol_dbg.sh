cd $GRAFT_REPO_ROOT
for v in 1 1; do HS_GEMM64=$v timeout 300 python tools/gpu/chol_det.py; done
timeout 1200 python -m pytest tests -m gpu -q -k "chol or factor or spd or potf or gemm or substitution or not_spd or singular or finite or oz or cyclic or group or fullsize" 2>&1 | grep -E "FAILED|passed|failed|Error|assert" | head -40
for k in 1 2; do for v in 1 0; do
echo "== HS_GEMM64=$v"; HS_GEMM64=$v timeout 300 python tools/chol_bench.py --n 32768 --b 512 --slices 0 8 --reps 2 2>&1 | grep -v "^chol " ; done; done
