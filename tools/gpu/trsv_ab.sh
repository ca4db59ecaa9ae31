#!/bin/bash
# substitution timings (forward + backward) at three sizes
for nb in "32768 512" "16384 256" "8192 128"; do
  set -- $nb
  timeout 300 python tools/trsv_bench.py --n $1 --b $2 --reps 10 2>&1 | tail -1
done
