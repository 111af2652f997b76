#!/bin/bash
# quick GPU iteration: all GPU tests, phase timings, short bench, full-solve timings
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
for n in 1023 2047 4095; do FD_PHASE_TIMING=1 timeout 60 python tools/prof_c1.py --steps 3 --n $n 2>&1 | grep "phase us" | tail -1; done
timeout 300 python bench.py --steps 300 --warmup 5 --no-cpu > gpurun_out/bench.log 2>&1; echo "bench rc=$?"; cut -c1-400 gpurun_out/bench.log
timeout 600 python tools/solve_timing.py c0 c2 c3 c4 > gpurun_out/solve_timing.log 2>&1; echo "solves rc=$?"; cat gpurun_out/solve_timing.log
