cd $GRAFT_REPO_ROOT
timeout 600 ncu --set full --import-source on --clock-control none -k regex:diag128 -s 8 -c 1 -o gpurun_out/diag128_full -f python tools/chol_bench.py --n 4096 --b 512 --slices 0 --reps 0 > gpurun_out/diag_ncu.log 2>&1
