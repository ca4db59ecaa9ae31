set -x
cd $GRAFT_REPO_ROOT
for rep in 1 2; do
for v in "8:" "0:1:8" "0:1:16" "8:1:8" "0:2:64" "0:2:128" "8:2:128" "0:2:48" "0:1:24"; do
  pf=${v%%:*}; keep=${v#*:}
  echo "== pf=$pf keep=$keep"
  HS_SYMV_PF_SLABS=$pf HS_SYMV_KEEP=$keep timeout 300 python tools/cg_iter_bench.py 32768 128 400 2>/dev/null | grep "events"
done
done
