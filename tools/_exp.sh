HS_SLAB_TRACE=1 timeout 300 python tools/profile_pass.py --which 1 --batch 32 > gpurun_out/strace.txt 2>&1
HS_SLAB_TRACE=1 timeout 300 python tools/profile_pass.py --which 1 --batch 16 >> gpurun_out/strace.txt 2>&1
HS_SLAB_TRACE=1 timeout 300 python tools/profile_pass.py --which 1 --batch 1 >> gpurun_out/strace.txt 2>&1
