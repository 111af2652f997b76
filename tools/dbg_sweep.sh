#!/bin/bash
# component costs of the persistent c1 apply: FD_DBG bits skip parts (timing only, results invalid;
# needs a build with -DFD_DIAG=1)
# 1: phase-3 output stores  2: phase-1 yhat stores  8: phase-1 FFT  16: phase-1 sweep  32: phase-3 FFT  64: phase-3 sweep
for d in 0 1 2 8 16 32 64 24 96; do echo -n "dbg $d: "; FD_DBG=$d FD_PHASE_TIMING=1 timeout 60 python tools/prof_c1.py --steps 3 2>&1 | grep "phase us" | tail -1; done
echo -n "rsws: "; FD_RSWS=1 FD_PHASE_TIMING=1 timeout 60 python tools/prof_c1.py --steps 3 2>&1 | grep "phase us" | tail -1
