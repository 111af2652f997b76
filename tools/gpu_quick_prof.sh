#!/bin/bash
./tools/gpu_quick.sh
python tools/prof_c1.py > gpurun_out/prof_plain.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:persist -s 2 -c 1 -o gpurun_out/prof_c1_cur -f python tools/prof_c1.py --steps 3 > gpurun_out/ncu_cur.log 2>&1
echo done
