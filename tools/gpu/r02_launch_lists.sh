#!/bin/bash
# launch lists (ncu, serialized, cold per launch) of the Cholesky n=32768 and a CG run
cd $GRAFT_REPO_ROOT
O=gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum,launch__grid_size --clock-control none --csv --log-file $O/r02_chol_launches.csv python tools/prof_run.py chol --n 32768 --b 512 > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/r02_cg_launches.csv python tools/prof_run.py cg --n 32768 --b 128 --iters 12 > /dev/null 2>&1
ls -la $O/r02_*launches.csv
