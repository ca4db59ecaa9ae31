#!/bin/bash
timeout 1500 compute-sanitizer --tool racecheck --racecheck-report hazard --print-limit 100000 python tools/gpu/sanitize_odd.py > /tmp/rc_odd.txt 2>&1
python - <<'PY'
import re, collections
txt=open('/tmp/rc_odd.txt').read()
cnt=collections.Counter()
for b_ in txt.split('Error: Potential')[1:]:
    kind=b_.split(' hazard')[0].strip()
    locs=re.findall(r'(Read|Write) Thread \([0-9,]+\) at ([^\n]*?) in ([a-z_]+\.cu[h]?:\d+)', b_)
    cnt[(kind,)+tuple((l[0], l[1].split('(')[0].split('+')[0][-40:], l[2]) for l in locs)]+=1
for k,v in cnt.most_common(30): print(v,k)
print([l for l in txt.splitlines() if 'SUMMARY' in l or l.startswith('cg ') or l.startswith('simt')])
PY
timeout 900 compute-sanitizer --tool memcheck python tools/gpu/sanitize_odd.py 2>&1 | tail -3
