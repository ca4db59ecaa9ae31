#!/bin/bash
for w in cg dist; do
  timeout 1200 compute-sanitizer --tool racecheck --racecheck-report hazard --print-limit 100000 python tools/gpu/sanitize_more.py $w > /tmp/rc_$w.txt 2>&1
  echo "== $w"
  python - $w <<'PY'
import re, collections, sys
txt=open('/tmp/rc_%s.txt' % sys.argv[1]).read()
cnt=collections.Counter()
for b_ in txt.split('Error: Potential')[1:]:
    kind=b_.split(' hazard')[0].strip()
    locs=re.findall(r'(Read|Write) Thread \([0-9,]+\) at ([^\n]*?) in ([a-z_]+\.cu[h]?:\d+)', b_)
    cnt[(kind,)+tuple((l[0], l[1].split('(')[0].split('+')[0][-40:], l[2]) for l in locs)]+=1
for k,v in cnt.most_common(30): print(v,k)
print([l for l in txt.splitlines() if 'SUMMARY' in l or l.startswith('cg ') or l.startswith('dist ')])
PY
done
