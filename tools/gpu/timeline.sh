cd $GRAFT_REPO_ROOT
for v in "HS_CG_TAIL_LAUNCH=3" "HS_CG_TAIL_LAUNCH=0"; do
  echo "== $v"; env $v timeout 300 python tools/cg_timeline.py 32768 128 200 2
done > gpurun_out/timeline.txt 2>&1
