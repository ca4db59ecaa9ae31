#!/bin/bash
for k in 1 2; do for v in 0 1; do
  echo "== HS_GEMM64_BULK=$v"; HS_GEMM64_BULK=$v timeout 300 python tools/chol_bench.py --n 32768 --b 512 --slices 0 --reps 5 2>&1 | tail -1
done; done
HS_GEMM64_BULK=1 REPS=3 timeout 600 python tools/gpu/pollute_check.py 2>&1 | grep -v NCCL
bash tools/gpu/gemm64_ncu.sh
python tools/ncu_keymetrics.py gpurun_out/r02_gemm64_big.ncu-rep gpurun_out/r02_ncu_gemm64_big_fenced.json > /dev/null
