cd $GRAFT_REPO_ROOT
timeout 300 python tools/diag_timing.py > gpurun_out/diag_timing.txt 2>&1
HS_CHOL_TIMING=1 timeout 300 python tools/chol_bench.py --n 32768 --b 512 --slices 0 --reps 2 > gpurun_out/chol_timing.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q -k "chol or factor or spd or potf or substitution or not_spd or singular or finite or oz or cyclic or group or fullsize" 2>&1 | tail -4 > gpurun_out/chol_tests.txt
