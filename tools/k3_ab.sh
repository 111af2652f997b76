#!/bin/bash
# A/B of the N = 1024 solve kernels: FD_RS32=0 (lockstep rsolve.cu) vs 1 (rsolve32.cu)
# c1 bench value + per-phase stamps; run from the repo root on the GPU box.
for m in 0 1; do
  echo "== FD_RS32=$m"
  FD_RS32=$m FD_PHASE_TIMING=1 python tools/prof_c1.py --steps 3 2>&1 | tail -2
  FD_RS32=$m python bench.py --steps 200 --warmup 5 --no-cpu --no-solve 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('ms', d['ms_per_step']*1e3, 'us  frac', d['roofline']['frac'], 'check', d.get('check'))"
done
