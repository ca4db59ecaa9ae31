"""SASS inventory of libhsolve_cuda.so: per kernel, the count of the
instructions that prove which hardware path it runs on (B200_PROFILING.md):

  DMMA       FP64 tensor-core MMA (mma.sync .f64)
  UTCIMMA    tcgen05.mma kind::i8 (5th-gen tensor cores, INT8)
  UTCBAR     tcgen05.commit -> mbarrier
  LDTM       tcgen05.ld (TMEM -> registers)
  UTMALDG    TMA tensor load (cp.async.bulk.tensor)
  UBLKCP     TMA bulk copy (cp.async.bulk)
  UBLKRED    TMA bulk reduce (cp.reduce.async.bulk)
  UBLKPF     bulk L2 prefetch (cp.async.bulk.prefetch.L2)
  SYNCS      mbarrier arrive / wait (SYNCS.*)
  DFMA       scalar FP64 FMA

    python tools/sass_inventory.py [--so path] [--out profiles/r02_sass_inventory.txt]
"""
from __future__ import annotations

import argparse
import json
import os
import re
import subprocess
from collections import Counter, defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OPS = ["DMMA", "UTCIMMA", "UTCQMMA", "UTCHMMA", "UTCBAR", "LDTM", "STTM", "UTMALDG", "UTMASTG",
       "UBLKCP", "UBLKRED", "UBLKPF", "SYNCS", "DFMA", "DADD", "DMUL"]


def demangle(names):
    out = subprocess.run(["c++filt"], input="\n".join(names), capture_output=True, text=True)
    return out.stdout.splitlines()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--so", default=os.path.join(ROOT, "paper_2605_13209_b200", "libhsolve_cuda.so"))
    ap.add_argument("--out", default="")
    args = ap.parse_args()
    sass = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-sass", args.so],
                          capture_output=True, text=True, check=True).stdout
    counts: dict[str, Counter] = defaultdict(Counter)
    arch = set()
    cur = None
    for ln in sass.splitlines():
        m = re.match(r"\s*Function : (\S+)", ln)
        if m:
            cur = m.group(1)
            continue
        m = re.search(r"arch = (sm_\w+)", ln)
        if m:
            arch.add(m.group(1))
        if cur is None:
            continue
        m = re.match(r"\s*/\*[0-9a-f]+\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)", ln)
        if m:
            op = m.group(1)
            for k in OPS:
                if op == k or op.startswith(k + "."):
                    counts[cur][k] += 1
    names = sorted(counts)
    pretty = dict(zip(names, demangle(names)))
    rows = []
    for n in names:
        c = {k: v for k, v in counts[n].items() if v}
        if any(k not in ("DFMA", "DADD", "DMUL") for k in c) or c.get("DFMA", 0) > 0:
            rows.append((pretty[n], c))
    lines = [f"SASS inventory of {os.path.relpath(args.so, ROOT)} (cuobjdump -sass; arch "
             f"{', '.join(sorted(arch))})", ""]
    for name, c in sorted(rows, key=lambda r: r[0]):
        short = re.sub(r"\(.*", "", name)
        lines.append(f"{short:60s} " + " ".join(f"{k}={c[k]}" for k in OPS if c.get(k)))
    text = "\n".join(lines)
    print(text)
    if args.out:
        with open(args.out, "w") as f:
            f.write(text + "\n")
        with open(os.path.splitext(args.out)[0] + ".json", "w") as f:
            json.dump({"arch": sorted(arch), "kernels": {re.sub(r"\(.*", "", n): c
                                                          for n, c in rows}}, f, indent=1)


if __name__ == "__main__":
    main()
