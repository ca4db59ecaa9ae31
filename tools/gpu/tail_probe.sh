cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "cg" > gpurun_out/tp_tests.log 2>&1; echo rc=$? >> gpurun_out/tp_tests.log
for k in 1 2; do
for v in "HS_CG_TAIL=0" "HS_CG_TAIL_LAUNCH=0" "HS_CG_TAIL_LAUNCH=3"; do
  env $v timeout 300 python bench.py --steps 200 --warmup 10 --no-secondary --no-cpu-baseline --no-anchor --no-e2e > gpurun_out/tp_$v.$k.json 2>gpurun_out/tp_$v.err
done
done
HS_CG_TAIL_LAUNCH=0 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 120 --csv --log-file gpurun_out/tail_launches.csv python bench.py --steps 20 --warmup 3 --no-secondary --no-cpu-baseline --no-anchor --no-e2e > /dev/null 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:cg_tail -s 5 -c 1 -o gpurun_out/tail_full python bench.py --steps 20 --warmup 3 --no-secondary --no-cpu-baseline --no-anchor --no-e2e > /dev/null 2>&1
