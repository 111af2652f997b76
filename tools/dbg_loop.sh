#!/bin/bash
# Partition robustness scan of the fused solve: the 5 x 1023^2 batch against the oracle under
# many row partitions (FD_TAU0 / FD_TAU2 move the range boundaries).  Prints BAD [] when all match.
for t2 in 0.0 0.3 0.6; do for t0 in 0 2 3 4 5 6 8 10; do
  echo -n "tau2=$t2 tau0=$t0: "; FD_TAU2=$t2 FD_TAU0=$t0 timeout 300 python tools/dbg_tau.py ${1:-1023} 2>/dev/null | grep BAD
done; done
