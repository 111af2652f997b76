#!/bin/bash
# bench lines + launch list + full capture of the dominant kernel (one GPU)
mkdir -p gpurun_out
timeout 600 python bench.py > gpurun_out/bench_full.log 2>&1; echo "bench rc=$?"
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.log 2>&1; echo "ref rc=$?"
timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu --no-solve > gpurun_out/bench_short.log 2>&1 && \
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench.csv \
    python bench.py --steps 20 --warmup 3 --no-cpu --no-solve > gpurun_out/ncu_launch.log 2>&1; echo "ncu1 rc=$?"
timeout 600 bash tools/ncu_c1.sh; echo "ncu2 rc=$?"
timeout 900 python tools/solve_timing.py c0 c2 c3 c4 > gpurun_out/solve_timing.log 2>&1; echo "solves rc=$?"
