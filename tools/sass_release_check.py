"""Flag mbarrier consumer releases that can retire before the shared-memory
reads they release have returned.

For every `SYNCS.ARRIVE.TRANS64.A1T0` (a consumer's arrive on an `empty`
barrier) in a kernel's SASS, collect the destination registers of the `LDS`
issued since the previous barrier operation, and report the arrive if any of
them is read AFTER it (the load may still be in flight when the producer
refills the stage) with no `MEMBAR` in between. Usage:
    python tools/sass_release_check.py paper_2605_13209_b200/libhsolve_cuda.so
"""
import re
import subprocess
import sys

INS = re.compile(r"/\*[0-9a-f]{4,}\*/\s+(.*?)\s*;")


def regs(tok, width):
    m = re.match(r"R(\d+)", tok)
    if not m:
        return []
    base = int(m.group(1))
    return [f"R{base + k}" for k in range(width)]


def width_of(op):
    if ".128" in op:
        return 4
    if ".64" in op:
        return 2
    return 1


def check(lines):
    ins = [INS.search(l).group(1) for l in lines if INS.search(l)]
    bad = []
    for k, s in enumerate(ins):
        if "SYNCS.ARRIVE.TRANS64.A1T0" not in s:
            continue
        pending = set()
        fenced = False
        for b in range(k - 1, max(k - 400, -1), -1):
            t = ins[b]
            if "SYNCS" in t or "BAR.SYNC" in t or re.match(r"(@\S+\s+)?BRA", t):
                break
            if "MEMBAR" in t and not pending:
                fenced = True
            if re.search(r"\bLDS(\.\w+)*\s", t) and not fenced:
                op, rest = t.split(None, 1) if not t.startswith("@") else t.split(None, 2)[1:]
                dst = rest.split(",")[0].strip()
                pending.update(regs(dst, width_of(op)))
        if not pending:
            continue
        for f in range(k + 1, min(k + 400, len(ins))):
            t = ins[f]
            if re.match(r"(@\S+\s+)?(BRA|EXIT|RET)", t) or "MEMBAR" in t:
                break
            parts = t.split(None, 1)
            if len(parts) < 2:
                continue
            ops = [o.strip() for o in parts[1].split(",")]
            srcs = set()
            for o in ops[1:]:
                for r in re.findall(r"R\d+", o):
                    srcs.add(r)
            hit = pending & srcs
            if hit:
                bad.append((k, s, t, sorted(hit)[:4]))
                break
            dst = ops[0] if ops else ""
            for r in re.findall(r"R\d+", dst):
                pending.discard(r)
    return bad


def main(so):
    txt = subprocess.run(["cuobjdump", "-sass", so], capture_output=True, text=True).stdout
    funcs = re.split(r"\n\s*Function : ", txt)
    n_bad = 0
    for f in funcs[1:]:
        name = f.split("\n", 1)[0].strip()
        bad = check(f.split("\n"))
        if bad:
            n_bad += 1
            k, s, t, r = bad[0]
            print(f"{name}: {len(bad)} release(s) ahead of pending LDS, e.g. '{s}' then '{t}' reads {r}")
    print(f"{n_bad} kernel(s) flagged")
    return n_bad


if __name__ == "__main__":
    sys.exit(1 if main(sys.argv[1]) else 0)
