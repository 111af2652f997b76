#!/bin/bash
# A/B of alternative library builds on full solves: paper_2509_23180_b200/libfftddm_b200.so.<tag>
L=paper_2509_23180_b200/libfftddm_b200.so
for tag in "$@"; do
  cp $L.$tag $L
  echo "== $tag"; timeout 300 python tools/solve_timing.py c0 c2 c3 --reps 3 2>&1 | python -c "
import json, sys
for l in sys.stdin:
    if l.startswith('{'):
        d = json.loads(l); print(d['config'], d['iterations'], round(d['wall_s'] * 1e3, 2), 'ms', d.get('rel_l2_exact'))"
done
