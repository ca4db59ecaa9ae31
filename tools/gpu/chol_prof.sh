cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests -m gpu -x -q -k "chol or factor or spd or potf or gemm or substitution or not_spd or singular or finite or oz or cyclic or group or fullsize" 2>&1 | tail -4 > gpurun_out/chol_tests.txt
for k in 1 2; do for v in 1 0; do
echo "== HS_GEMM64=$v"; HS_GEMM64=$v HS_CHOL_TIMING=1 timeout 300 python tools/chol_bench.py --n 32768 --b 512 --slices 0 --reps 2 2>&1 | grep -v "^chol " ; done; done > gpurun_out/chol_ab.txt 2>&1
HS_CHOL_TIMING=1 timeout 300 python tools/chol_bench.py --n 32768 --b 512 --slices 0 --reps 1 > gpurun_out/chol_timing.txt 2>&1
