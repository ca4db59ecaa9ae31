cd $GRAFT_REPO_ROOT
for v in 1 0; do
HS_CHOL_PAIRS=$v timeout 900 ncu --metrics gpu__time_duration.sum,launch__grid_size,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:gemm_dmma --csv --log-file gpurun_out/chol_pairs_$v.csv python tools/prof_run.py chol --n 32768 --b 512 > /dev/null 2>&1
done
