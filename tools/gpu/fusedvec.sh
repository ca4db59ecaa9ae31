cd $GRAFT_REPO_ROOT
for v in 1 0; do
  echo "== HS_CG_FUSED_VEC=$v"; HS_CG_FUSED_VEC=$v timeout 300 python tools/cg_timeline.py 32768 128 200 1 2>&1 | grep -v "per-CTA\|fused\|progressive"
done
for k in 1 2; do for v in 1 0; do
  echo "== HS_CG_FUSED_VEC=$v"; HS_CG_FUSED_VEC=$v timeout 300 python tools/cg_iter_bench.py 32768 128 400 2>/dev/null | grep -E "events|converging"
done; done
HS_CG_FUSED_VEC=1 timeout 900 python -m pytest tests -m gpu -q -k "cg" 2>&1 | tail -2
