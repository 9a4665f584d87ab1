# ncu captures behind profiles/round2 (run on the GPU box from the repo root)
set -x
mkdir -p gpurun_out/r2
NCU="ncu --clock-control none"
# 1. launch list of the bench step (2 timed steps, B = 32)
timeout 900 $NCU --metrics gpu__time_duration.sum --csv --log-file gpurun_out/r2/launches_b32.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu > gpurun_out/r2/bench_under_ncu.log 2>&1
# 2. window pass, B = 32 (the time_kernel launch after one solve's 38 graph launches)
timeout 900 $NCU --set full --import-source on -k regex:hs_slab_kernel -s 38 -c 1 -f -o gpurun_out/r2/slab_b32 \
    python tools/profile_pass.py --which 1 --batch 32 > gpurun_out/r2/slab.log 2>&1
# 3. tcgen05 full pass, B = 32
timeout 900 $NCU --set full --import-source on -k regex:hs_umma_kernel -s 4 -c 1 -f -o gpurun_out/r2/umma_b32 \
    python tools/profile_pass.py --which 0 --batch 32 > gpurun_out/r2/umma.log 2>&1
# 4. tcgen05 spot-chunked full pass at config 4 (N = 1000, one hologram)
timeout 900 $NCU --set full --import-source on -k regex:hs_umma_kernel -s 3 -c 1 -f -o gpurun_out/r2/umma_n1000 \
    python tools/profile_pass.py --which 0 --batch 1 --spots 1000 > gpurun_out/r2/umma1000.log 2>&1
# 5. B = 1 launch list (single-hologram latency)
timeout 600 $NCU --metrics gpu__time_duration.sum --csv --log-file gpurun_out/r2/launches_b1.csv \
    python tools/latency_probe.py --reps 1 > /dev/null 2>&1
