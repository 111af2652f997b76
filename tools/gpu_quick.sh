#!/bin/bash
# quick GPU iteration: parity tests + phase timings + bench (used via gpurun)
timeout 600 python -m pytest tests -m gpu -q -x -k "not slow" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
for n in 1023 2047 4095; do FD_PHASE_TIMING=1 timeout 60 python tools/prof_c1.py --steps 2 --n $n 2>&1 | tail -2; done > gpurun_out/phase.log 2>&1
timeout 300 python bench.py --steps 200 --warmup 5 --no-cpu > gpurun_out/bench.log 2>&1; echo "bench rc=$?"
