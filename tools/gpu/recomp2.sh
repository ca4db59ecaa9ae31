cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests -m gpu -q -k "cg or symv or fullsize or reference" 2>&1 | tail -3
for k in 1 2; do for v in 1 0; do
  echo "== HS_CG_RECOMP2=$v"
  HS_CG_RECOMP2=$v timeout 300 python tools/cg_iter_bench.py 32768 128 400 2>/dev/null | grep -E "events|converging"
done; done
