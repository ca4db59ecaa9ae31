# progressive SYMV/finalize: GPU tests of the CG paths, then A/B against the
# memory-order walk (HS_CG_PROG=0), interleaved
cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests -m gpu -x -q -k "symv or cg or ledger or multirank or group or smoke" 2>&1 | tail -15
for rep in 1 2; do
for v in 1 0; do
  echo "== HS_CG_PROG=$v"
  HS_CG_PROG=$v timeout 300 python tools/cg_iter_bench.py 32768 128 400 2>/dev/null | grep -E "events|hs_symv|converging"
done
done
