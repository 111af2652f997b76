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
# launch 30 of the bench's rotating-buffer loop (the `traffic` of the bench line) and one N = 4096 apply
timeout 300 ncu --set full --clock-control none -k regex:"rsolve" -s 30 -c 1 -f -o gpurun_out/prof_c1_loop \
    python bench.py --steps 40 --warmup 5 --no-cpu --no-solve > gpurun_out/ncu_loop.log 2>&1; echo "ncu3 rc=$?"
timeout 300 ncu --set full --clock-control none --import-source on -k regex:"rsolve" -s 2 -c 1 -f -o gpurun_out/prof_n4095 \
    python tools/prof_c1.py --n 4095 --steps 3 > gpurun_out/ncu_n4095.log 2>&1; echo "ncu4 rc=$?"
for n in 1023 2047 4095; do FD_PHASE_TIMING=1 timeout 60 python tools/prof_c1.py --steps 4 --n $n 2>&1 | grep "phase us" | tail -1; done > gpurun_out/phase_times.log
timeout 900 python tools/solve_timing.py c0 c2 c3 c4 > gpurun_out/solve_timing.log 2>&1; echo "solves rc=$?"
timeout 900 python tools/solve_timing.py c0 c2 c3 c4 --steklov >> gpurun_out/solve_timing.log 2>&1; echo "solves-if rc=$?"
timeout 900 python tools/solve_timing.py c2 c4 --assemble --reps 3 >> gpurun_out/solve_timing.log 2>&1; echo "solves-asm rc=$?"
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
