rm -f gpurun_out/cpc.txt
for c in 0 1 2 4 8 16; do echo "cpc $c" >> gpurun_out/cpc.txt; HS_SLAB_CPC=$c timeout 300 python tools/ab_time.py >> gpurun_out/cpc.txt 2>&1; done
