cd $GRAFT_REPO_ROOT
for k in 1 2; do
for v in 0 1; do
  echo "== HS_CHOL_SCHED=$v"
  HS_CHOL_SCHED=$v timeout 300 python tools/chol_bench.py --n 32768 --b 512 --slices 0 --reps 3
done
done > gpurun_out/chol_ab.txt 2>&1
HS_CHOL_SCHED=1 timeout 300 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "chol or factor or spd" >> gpurun_out/chol_ab.txt 2>&1
