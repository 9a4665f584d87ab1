# scratch driver for one gpurun experiment (the last one run is kept here)
for v in 0; do HS_SLAB_PIPE=$v timeout 300 python tools/ab_time.py; done > gpurun_out/ab4.txt 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:hs_slab_kernel -s 5 -c 1 -f -o gpurun_out/slab_r2b python tools/profile_pass.py --which 1 --batch 32 > gpurun_out/ncu_slab.log 2>&1
