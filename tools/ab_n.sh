#!/bin/bash
# A/B of library variants (paper_2509_23180_b200/libfftddm_b200.so.<tag>) at several transform
# lengths: per-phase stamps of the batched solve (5 rectangles of n x n).  Usage: ab_n.sh "n1 n2" tag...
ns=$1; shift
for tag in "$@"; do
  cp paper_2509_23180_b200/libfftddm_b200.so.$tag paper_2509_23180_b200/libfftddm_b200.so
  for n in $ns; do
    echo -n "== $tag n=$n: "; FD_PHASE_TIMING=1 timeout 60 python tools/prof_c1.py --steps 4 --n $n 2>&1 | grep "phase us" | tail -1 | cut -c14-190
  done
done
