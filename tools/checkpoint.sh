#!/bin/bash
# full GPU checkpoint: every GPU test (incl. slow full-size parity), per-N sweeps, bench
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu_all.log 2>&1; echo "pytest rc=$?"
for n in 255 511 1023 2047; do timeout 300 python tools/diag_m.py $n 1,17,40,700,1185; done > gpurun_out/diag_m.log 2>&1; echo "diag rc=$?"
timeout 300 python bench.py --steps 300 --warmup 5 > gpurun_out/bench_full.log 2>&1; echo "bench rc=$?"
timeout 300 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.log 2>&1; echo "ref rc=$?"
