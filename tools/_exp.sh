mkdir -p gpurun_out
HS_UMMA=1 timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_umma.txt 2>&1
tail -3 gpurun_out/pytest_gpu_umma.txt
HS_UMMA=1 timeout 300 python tools/profile_pass.py --which 0 --batch 32 --reps 20
