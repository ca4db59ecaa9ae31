cd $GRAFT_REPO_ROOT
timeout 900 compute-sanitizer --tool racecheck --racecheck-report all --kernel-regex kns=symv_slab python tools/gpu/sanitize_prog.py 2>&1 | grep -v "^=========     in \|^=========         " | head -60
