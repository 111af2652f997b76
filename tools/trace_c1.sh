FD_TRACE=70 timeout 60 python tools/prof_c1.py --steps 2 > gpurun_out/trace70.log 2>&1
FD_TRACE=0 timeout 60 python tools/prof_c1.py --steps 2 > gpurun_out/trace0.log 2>&1
FD_PHASE_TIMING=1 FD_PHASE_TIMING_CTA=1 timeout 60 python tools/prof_c1.py --steps 2 > gpurun_out/phase_cta.log 2>&1
