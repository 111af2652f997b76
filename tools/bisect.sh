#!/bin/bash
for d in 0 8 16 24 9; do echo "dbg=$d"; FD_DBG=$d FD_PHASE_TIMING=1 FD_PHASE_TIMING_CTA=1 timeout 60 python tools/prof_c1.py --steps 2 2>&1 | grep -E "phase|cta" | tail -8; done
