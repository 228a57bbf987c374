#!/usr/bin/env python
"""Mean per-iteration ms and per-class ms over iterations [lo, hi] of tools/probe.py outputs."""
import json
import sys

lo, hi = 6, 12
for f in sys.argv[1:]:
    rows = [json.loads(l) for l in open(f) if l.startswith('{"t"')]
    w = [r for r in rows if lo <= r['t'] <= hi]
    if not w:
        print(f, "no rows")
        continue
    tot = sum(r['ms'] for r in w) / len(w)
    cls = {}
    for r in w:
        for k, v in r['cls'].items():
            cls[k] = cls.get(k, 0) + v / len(w)
    dist = sum(r['dist'] for r in w) / len(w)
    print(f, round(tot, 2), {k: round(v, 2) for k, v in cls.items()}, "dist %.3g" % dist)
