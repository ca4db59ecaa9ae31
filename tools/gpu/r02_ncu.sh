# round-2 evidence: launch lists (CG iteration, Cholesky) and full captures of
# the progressive SYMV, the split-tile DMMA GEMMs and diag128
cd $GRAFT_REPO_ROOT
O=gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/r02_cg_launches.csv python tools/prof_run.py cg --n 32768 --b 128 --iters 12 > /dev/null 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,launch__grid_size --clock-control none --csv --log-file $O/r02_chol_launches.csv python tools/prof_run.py chol --n 32768 --b 512 > /dev/null 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:symv_slab -s 3 -c 1 -o $O/r02_symv_prog -f python tools/prof_run.py cg --n 32768 --b 128 --iters 6 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none -k regex:"gemm_dmma_kernel<64, 64>" -s 40 -c 1 -o $O/r02_gemm64 -f python tools/prof_run.py chol --n 16384 --b 512 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none -k regex:"gemm_dmma_kernel<64, 128>" -s 40 -c 1 -o $O/r02_gemm64x128 -f python tools/prof_run.py chol --n 16384 --b 512 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none -k regex:"gemm_dmma_kernel<128, 128>" -s 5 -c 1 -o $O/r02_gemm128 -f python tools/prof_run.py chol --n 16384 --b 512 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none -k regex:diag128 -s 20 -c 1 -o $O/r02_diag128 -f python tools/prof_run.py chol --n 16384 --b 512 > /dev/null 2>&1
ls -la $O/*.ncu-rep $O/r02_*.csv
