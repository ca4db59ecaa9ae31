cd $GRAFT_REPO_ROOT
free -g > gpurun_out/free.txt
for v in "HS_CG_TAIL=0" "HS_CG_TAIL_LAUNCH=0" "HS_CG_TAIL_LAUNCH=2" "HS_CG_TAIL_LAUNCH=3"; do
  env $v timeout 300 python bench.py --steps 200 --warmup 10 --no-secondary --no-cpu-baseline --no-anchor --no-e2e > gpurun_out/tp_$v.json 2>gpurun_out/tp_$v.err
done
HS_CG_TAIL_LAUNCH=0 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 120 --csv --log-file gpurun_out/tail_launches.csv python bench.py --steps 20 --warmup 3 --no-secondary --no-cpu-baseline --no-anchor --no-e2e > /dev/null 2>&1
HS_CG_TAIL=0 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 120 --csv --log-file gpurun_out/notail_launches.csv python bench.py --steps 20 --warmup 3 --no-secondary --no-cpu-baseline --no-anchor --no-e2e > /dev/null 2>&1
