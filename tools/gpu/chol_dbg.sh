cd $GRAFT_REPO_ROOT
for k in 1 2; do for v in 1 0; do
echo "== HS_OZ_U_HIPRI=$v"; HS_OZ_U_HIPRI=$v timeout 300 python tools/chol_bench.py --n 32768 --b 512 --slices 8 --reps 2 2>&1 | grep -v "^chol " ; done; done
timeout 600 python tools/chol_bench.py --n 131072 --b 512 --slices 0 8 --reps 1
timeout 600 python tools/chol_bench.py --n 16384 --b 512 --slices 0 8 --reps 2
timeout 600 python tools/chol_bench.py --n 32768 --b 256 --slices 0 --reps 2
HS_CHOL_PAIRS=0 timeout 600 python tools/chol_bench.py --n 32768 --b 256 --slices 0 --reps 2
timeout 1200 python -m pytest tests -m gpu -q 2>&1 | tail -3
