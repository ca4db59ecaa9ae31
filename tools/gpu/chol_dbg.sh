cd $GRAFT_REPO_ROOT
timeout 300 python tools/gpu/chol_det.py
for k in 1 2; do for v in 1 0; do
echo "== HS_CHOL_PANEL_OVERLAP=$v"; HS_CHOL_PANEL_OVERLAP=$v timeout 300 python tools/chol_bench.py --n 32768 --b 512 --slices 0 8 --reps 2 2>&1 | grep -v "^chol " ; done; done
timeout 1500 python -m pytest tests -m gpu -q -k "chol or factor or spd or potf or gemm or substitution or not_spd or singular or finite or oz or fullsize or split" 2>&1 | tail -2
