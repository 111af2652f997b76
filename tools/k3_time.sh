#!/bin/bash
# c1 apply time + phase stamps of library variants (no correctness check)
for v in "$@"; do
  cp paper_2509_23180_b200/libfftddm_b200.so.$v paper_2509_23180_b200/libfftddm_b200.so
  echo "== $v $(timeout 100 python tools/k3_check.py 2>&1 | grep 'c1 apply')"
  FD_PHASE_TIMING=1 timeout 60 python tools/prof_c1.py --steps 3 2>&1 | grep "phase us\] start" | tail -1
done
