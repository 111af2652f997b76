#!/bin/bash
# A/B of alternative library builds: paper_2509_23180_b200/libfftddm_b200.so.<tag>
for tag in "$@"; do
  cp paper_2509_23180_b200/libfftddm_b200.so.$tag paper_2509_23180_b200/libfftddm_b200.so
  echo "== $tag"; FD_PHASE_TIMING=1 timeout 60 python tools/prof_c1.py --steps 3 2>&1 | grep "phase us" | tail -1
  timeout 120 python bench.py --steps 300 --no-cpu --no-solve | python -c "import json,sys; l=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('ms', l['ms_per_step'])"
done
