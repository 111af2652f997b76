#!/bin/bash
# full Nsight Compute capture of one persistent c1 apply (after a clean run)
python tools/prof_c1.py > gpurun_out/prof_plain.log 2>&1 || exit 1
ncu --set full --clock-control none --import-source on -k regex:"persist|rsolve" -s 3 -c 1 -f -o gpurun_out/prof_c1_cur \
    python tools/prof_c1.py --steps 4 > gpurun_out/ncu_cur.log 2>&1; echo "ncu rc=$?"
