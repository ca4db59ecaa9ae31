cd $GRAFT_REPO_ROOT
for v in "1 1" "1 0" "0 0"; do
  set -- $v
  echo "== HS_CG_PROG=$1 HS_CG_FUSED_UPDATE=$2"
  HS_CG_PROG=$1 HS_CG_FUSED_UPDATE=$2 timeout 300 python tools/cg_timeline.py 32768 128 200 1 2>&1 | grep -v "per-CTA\|fused\|progressive"
done
for v in "1 1" "1 0" "0 0" "1 1" "1 0" "0 0"; do
  set -- $v
  echo "== HS_CG_PROG=$1 HS_CG_FUSED_UPDATE=$2"
  HS_CG_PROG=$1 HS_CG_FUSED_UPDATE=$2 timeout 300 python tools/cg_iter_bench.py 32768 128 400 2>/dev/null | grep -E "events|converging"
done
timeout 900 python -m pytest tests -m gpu -x -q -k "symv or cg or ledger or multirank or group" 2>&1 | tail -4
