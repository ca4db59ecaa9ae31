cd $GRAFT_REPO_ROOT
for v in 0 1; do
  HS_CG_PROG=$v timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_bytes.sum --clock-control none -k regex:"symv|finalize|vec" -c 60 --csv \
     python tools/cg_iter_bench.py 32768 128 20 > gpurun_out/prog_ncu_$v.csv 2>/dev/null
done
