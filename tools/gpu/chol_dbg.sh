cd $GRAFT_REPO_ROOT
for k in 1 2; do for v in 0 2; do
echo "== HS_GEMM_TILE=$v"; HS_GEMM_TILE=$v timeout 300 python tools/chol_bench.py --n 32768 --b 512 --slices 0 --reps 2 2>&1 | grep -v "^chol " ; done; done
