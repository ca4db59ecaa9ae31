cd $GRAFT_REPO_ROOT
for k in 1 2 3; do for v in 1 2; do
echo "== HS_GEMM64=$v"; HS_GEMM64=$v timeout 300 python tools/chol_bench.py --n 32768 --b 512 --slices 8 --reps 2 2>&1 | grep -v "^chol " ; done; done
