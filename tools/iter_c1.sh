#!/bin/bash
# quick iteration: correctness probe, phase timing, CTA trace, bench (c1)
timeout 120 python tools/diag_modes.py > gpurun_out/diag.log 2>&1; echo "diag rc=$?"
FD_PHASE_TIMING=1 FD_PHASE_TIMING_CTA=1 timeout 60 python tools/prof_c1.py --steps 3 > gpurun_out/ws_phase.log 2>&1; echo "prof rc=$?"
FD_TRACE=70 timeout 60 python tools/prof_c1.py --steps 2 > gpurun_out/trace70.log 2>&1
timeout 120 python bench.py --steps 500 --warmup 5 --no-cpu > gpurun_out/bench.log 2>&1; echo "bench rc=$?"
[ "$1" = "ncu" ] && bash tools/ncu_c1.sh
[ "$1" = "test" ] && { timeout 300 python -m pytest tests -m gpu -q -x -k "not slow" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; }
true
