cd $GRAFT_REPO_ROOT
timeout 600 ncu --metrics gpu__time_duration.sum,launch__grid_size --clock-control none -k regex:gemm_dmma --csv --log-file gpurun_out/g64_list.csv python tools/prof_run.py chol --n 16384 --b 512 > /dev/null 2>&1
IDX=$(python3 - <<'PY'
import csv, collections
rows=[r for r in csv.reader(open('gpurun_out/g64_list.csv')) if len(r)>10]
h=rows[0]; ii=h.index('ID'); mi=h.index('Metric Name'); vi=h.index('Metric Value')
g=collections.defaultdict(dict)
for r in rows[1:]: g[int(r[ii])][r[mi]]=float(r[vi].replace(',',''))
ids=sorted(g); best=max(ids, key=lambda i: g[i]['launch__grid_size'])
print(ids.index(best))
PY
)
echo "skip=$IDX"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:gemm_dmma -s $IDX -c 1 -o gpurun_out/r02_gemm64_big -f python tools/prof_run.py chol --n 16384 --b 512 > /dev/null 2>&1
ls -la gpurun_out/r02_gemm64_big.ncu-rep
