cd $GRAFT_REPO_ROOT
timeout 600 python tools/gpu/chol_dist_det.py 2>&1 | grep -v NCCL
HS_CHOL_PAIRS=0 timeout 600 python tools/gpu/chol_dist_det.py 2>&1 | grep -v NCCL | sed 's/^/nopairs /'
timeout 1500 python -m pytest tests -m gpu -q -k "group or multirank or dist or cyclic or ledger" 2>&1 | tail -2
for v in 1 0; do
  HS_CHOL_PAIRS=$v timeout 900 python bench.py --dist --steps 50 --warmup 3 --no-e2e --no-cpu-baseline --chol-reps 2 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); sc=d['secondary']; print('pairs=$v dist chol ms', sc.get('ms_per_factor'), sc.get('value'), sc.get('error'))"
done
