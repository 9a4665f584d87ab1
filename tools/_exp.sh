mkdir -p gpurun_out
HS_UMMA=1 timeout 600 ncu --set full --import-source on --clock-control none -k regex:hs_umma -s 2 -c 1 -o gpurun_out/umma32 python tools/profile_pass.py --which 0 --batch 32 --reps 1 > gpurun_out/ncu_umma.log 2>&1
tail -3 gpurun_out/ncu_umma.log
