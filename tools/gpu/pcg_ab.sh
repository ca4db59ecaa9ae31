#!/bin/bash
for v in 0 1; do
  echo "== HS_REFINE_PCG=$v"
  HS_REFINE_PCG=$v timeout 600 python tools/refine_bench.py --n 32768 --b 512 --slices 4 5 6 --reps 2 2>&1 | grep slices
done
HS_REFINE_PCG=1 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_multirank_gpu.py -q -m gpu -k refine 2>&1 | tail -2
echo "== n=131072, PCG"
HS_REFINE_PCG=1 timeout 900 python tools/refine_bench.py --n 131072 --b 512 --slices 4 --reps 1 2>&1 | grep slices
