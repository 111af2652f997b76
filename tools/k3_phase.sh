#!/bin/bash
# K3 bring-up on the GPU: correctness + c1 apply time + per-phase timestamps
for v in "$@"; do
  cp paper_2509_23180_b200/libfftddm_b200.so.$v paper_2509_23180_b200/libfftddm_b200.so
  echo "== $v"
  timeout 200 python tools/k3_check.py 2>&1 | tail -3
  FD_PHASE_TIMING=1 timeout 60 python tools/prof_c1.py --steps 3 2>&1 | grep "phase us" | tail -1
done
