#!/bin/bash
# full GPU validation: tests, smoke, bench line, Cholesky timings (single / dist world 1 / n=131072)
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/val_pytest.txt 2>&1; echo "pytest exit $?" >> gpurun_out/val_pytest.txt
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/val_smoke.txt 2>&1
timeout 600 python bench.py > gpurun_out/val_bench.json 2> gpurun_out/val_bench.err
timeout 600 python bench.py --impl reference > gpurun_out/val_bench_ref.json 2> gpurun_out/val_bench_ref.err
timeout 300 python tools/chol_bench.py --n 32768 --b 512 --slices 0 8 --reps 5 > gpurun_out/val_chol.txt 2>&1
timeout 900 python bench.py --dist --steps 50 --warmup 3 --no-e2e --no-cpu-baseline --chol-reps 2 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); sc=d['secondary']; print('dist chol ms', sc.get('ms_per_factor'), sc.get('value'), sc.get('error'))" >> gpurun_out/val_chol.txt 2>&1
timeout 900 python tools/chol_bench.py --n 131072 --b 512 --slices 0 --reps 1 >> gpurun_out/val_chol.txt 2>&1
bash tools/gpu/trsv_ab.sh >> gpurun_out/val_chol.txt 2>&1
