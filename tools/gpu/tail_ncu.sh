cd $GRAFT_REPO_ROOT
timeout 600 ncu --set full --import-source on --cache-control none --clock-control none -k regex:cg_tail -s 10 -c 1 -o gpurun_out/tail_full_warm python bench.py --steps 30 --warmup 3 --no-secondary --no-cpu-baseline --no-anchor --no-e2e > /dev/null 2>&1
HS_CG_TAIL=0 timeout 600 ncu --set full --import-source on --cache-control none --clock-control none -k regex:finalize -s 10 -c 1 -o gpurun_out/fin_full_warm python bench.py --steps 30 --warmup 3 --no-secondary --no-cpu-baseline --no-anchor --no-e2e > /dev/null 2>&1
