#!/bin/bash
# timing of c1 under FD_DBG experiment bits (results are NOT valid solves)
for d in "$@"; do
  echo "dbg=$d" >> gpurun_out/dbg.log
  FD_DBG=$d FD_PHASE_TIMING=1 timeout 60 python tools/prof_c1.py --steps 3 2>&1 | grep "fd phase" | tail -1 >> gpurun_out/dbg.log
done
