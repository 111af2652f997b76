#!/bin/bash
# Sweep the row-partition cost model (FD_TAU1, FD_TAU0) on c1: per-CTA phase
# times and the bench step time for each setting.  Usage: tau_sweep.sh "t1 t0" ...
cfgs=("$@")
[ ${#cfgs[@]} -eq 0 ] && cfgs=("1.2 4")
for cfg in "${cfgs[@]}"; do
    set -- $cfg
    echo "tau1=$1 tau0=$2" >> gpurun_out/tau.log
    FD_TAU1=$1 FD_TAU0=$2 FD_PHASE_TIMING=1 FD_PHASE_TIMING_CTA=1 timeout 60 python tools/prof_c1.py --steps 3 2>&1 | sed -n 5,8p >> gpurun_out/tau.log
    FD_TAU1=$1 FD_TAU0=$2 timeout 100 python bench.py --steps 300 --warmup 5 --no-cpu 2>/dev/null | grep -oE '"ms_per_step": [0-9.]+' >> gpurun_out/tau.log
done
