#!/bin/bash
for d in 0 32; do echo "dbg=$d"; FD_DBG=$d FD_PHASE_TIMING=1 timeout 60 python tools/prof_c1.py --steps 3 2>&1 | grep -E "phase" | tail -1; done
