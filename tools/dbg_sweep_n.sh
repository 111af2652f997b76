#!/bin/bash
# component-skip timings of the persistent solve at transform length n (default 4095); needs
# paper_2509_23180_b200/libfftddm_b200.so.diag (FD_DIAG_BUILD=1 build).  Results are invalid, times only.
# 1: phase-3 output stores  2: phase-1 yhat stores  8: phase-1 FFT  16: phase-1 sweep  32: phase-3 FFT  64: phase-3 sweep
n=${1:-4095}
cp paper_2509_23180_b200/libfftddm_b200.so /tmp/lib_prod.so
cp paper_2509_23180_b200/libfftddm_b200.so.diag paper_2509_23180_b200/libfftddm_b200.so
for d in 0 1 2 8 16 32 64 24 96; do echo -n "n=$n dbg $d: "; FD_DBG=$d FD_PHASE_TIMING=1 timeout 60 python tools/prof_c1.py --steps 3 --n $n 2>&1 | grep "phase us" | tail -1 | cut -c1-200; done
cp /tmp/lib_prod.so paper_2509_23180_b200/libfftddm_b200.so
