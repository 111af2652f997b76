#!/bin/bash
# bench + launch list + full capture of the dominant kernel (one GPU)
python bench.py > gpurun_out/bench_full.log 2>&1; echo "bench rc=$?"
python bench.py --impl reference --steps 5 --warmup 1 > gpurun_out/bench_ref.log 2>&1; echo "ref rc=$?"
python bench.py --steps 20 --warmup 3 --no-cpu > gpurun_out/bench_short.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench.csv \
    python bench.py --steps 20 --warmup 3 --no-cpu > gpurun_out/ncu_launch.log 2>&1; echo "ncu1 rc=$?"
python tools/prof_c1.py > gpurun_out/prof_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:persist -s 2 -c 1 -f -o gpurun_out/prof_persist_c1 \
    python tools/prof_c1.py --steps 3 > gpurun_out/ncu_full.log 2>&1; echo "ncu2 rc=$?"
timeout 600 python tools/solve_timing.py c0 c2 c3 > gpurun_out/solve_timing.log 2>&1; echo "solves rc=$?"
