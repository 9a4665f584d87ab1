# scratch driver for one gpurun experiment (the last one run is kept here)
for w in 0 2; do timeout 300 python tools/profile_pass.py --which $w --batch 32 --reps 20; done
