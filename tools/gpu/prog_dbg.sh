cd $GRAFT_REPO_ROOT
for rep in 1 2; do
for v in "0 0" "1 1" "1 17" "1 0"; do
  set -- $v
  echo "== HS_CG_PROG=$1 HS_PROG_DBG=$2"
  HS_CG_PROG=$1 HS_PROG_DBG=$2 timeout 300 python tools/cg_iter_bench.py 32768 128 300 2>/dev/null | grep -E "events|hs_symv"
done
done
