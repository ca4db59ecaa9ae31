# CG timeline (debug build tools/libhsolve_cuda_symvtiming.so): progressive
# SYMV vs the memory-order walk, then interleaved iteration timings
cd $GRAFT_REPO_ROOT
for v in 1 0; do
  echo "== HS_CG_PROG=$v"
  HS_CG_PROG=$v timeout 300 python tools/cg_timeline.py 32768 128 200 1 2>&1 | grep -v "per-CTA\|fused"
done
for k in 1 2; do for v in 1 0; do
  echo "== HS_CG_PROG=$v"
  HS_CG_PROG=$v timeout 300 python tools/cg_iter_bench.py 32768 128 400 2>/dev/null | grep -E "events|converging"
done; done
