#!/bin/bash
# per-phase / per-item timelines of the persistent c1 apply
for n in 1023 2047; do FD_PHASE_TIMING=1 FD_PHASE_TIMING_CTA=1 timeout 60 python tools/prof_c1.py --steps 3 --n $n; done > gpurun_out/phase.log 2>&1
FD_TRACE=70 FD_DBG=4 timeout 60 python tools/prof_c1.py --steps 2 > gpurun_out/trace70.log 2>&1
FD_TRACE=0 timeout 60 python tools/prof_c1.py --steps 2 > gpurun_out/trace0.log 2>&1
python tools/trace_solve.py c3 > gpurun_out/trace_c3.log 2>&1; rm -f gpurun_out/trace_c3.json
