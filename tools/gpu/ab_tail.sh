set -x
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_reference_fullsize.py tests/test_group_gpu.py tests/test_cpp_shim.py tests/test_gpu_check_finite.py -q -m gpu -rs > gpurun_out/t3.log 2>&1; echo rc=$? >> gpurun_out/t3.log
for k in 1 2 3; do
  for v in 0 1; do
    HS_CG_TAIL=$v timeout 300 python bench.py --steps 200 --warmup 10 --no-secondary --no-cpu-baseline --no-anchor --no-e2e > gpurun_out/ab_tail$v.$k.json 2>/dev/null
  done
done
