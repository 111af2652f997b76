#!/bin/bash
# round evidence (one GPU): full GPU suite, bench lines, launch list, full
# capture of the dominant kernel, full-solve timings (default, interface-only,
# device-assembled)
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_all.log 2>&1; echo "pytest rc=$?"
timeout 600 python bench.py > gpurun_out/bench_full.log 2>&1; echo "bench rc=$?"
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.log 2>&1; echo "ref rc=$?"
timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu --no-solve > gpurun_out/bench_short.log 2>&1 && \
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench.csv \
    python bench.py --steps 20 --warmup 3 --no-cpu --no-solve > gpurun_out/ncu_launch.log 2>&1; echo "ncu1 rc=$?"
timeout 600 bash tools/ncu_c1.sh; echo "ncu2 rc=$?"
timeout 900 python tools/solve_timing.py c0 c2 c3 c4 > gpurun_out/solve_timing.log 2>&1; echo "solves rc=$?"
timeout 900 python tools/solve_timing.py c0 c2 c3 c4 --steklov >> gpurun_out/solve_timing.log 2>&1; echo "solves-if rc=$?"
timeout 900 python tools/solve_timing.py c2 c4 --assemble --reps 3 >> gpurun_out/solve_timing.log 2>&1; echo "solves-asm rc=$?"
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
