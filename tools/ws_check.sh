#!/bin/bash
FD_PHASE_TIMING=1 timeout 60 python tools/prof_c1.py --steps 3 > gpurun_out/ws_phase.log 2>&1; echo "prof rc=$?"
timeout 120 python tools/diag_modes.py > gpurun_out/diag.log 2>&1; echo "diag rc=$?"
timeout 300 python -m pytest tests -m gpu -q -x -k "not slow" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
timeout 120 python bench.py --steps 500 --warmup 5 --no-cpu > gpurun_out/bench.log 2>&1; echo "bench rc=$?"
