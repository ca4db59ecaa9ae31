cd $GRAFT_REPO_ROOT
for k in 1 2; do for v in 1 2 0; do
echo "== HS_GEMM64=$v"; HS_GEMM64=$v timeout 300 python tools/chol_bench.py --n 32768 --b 512 --slices 0 --reps 2 2>&1 | grep -v "^chol " ; done; done
timeout 300 python tools/chol_bench.py --n 32768 --b 256 --slices 0 --reps 2 2>&1 | grep -v "^chol "
timeout 300 python tools/chol_bench.py --n 16384 --b 512 --slices 0 8 --reps 2 2>&1 | grep -v "^chol "
timeout 300 python tools/gpu/chol_det.py
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -3
