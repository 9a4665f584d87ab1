mkdir -p gpurun_out
rm -f gpurun_out/pp.txt
HS_UMMA=1 timeout 300 python tools/profile_pass.py --which 0 --batch 32 --reps 20 >> gpurun_out/pp.txt 2>&1
HS_UMMA=1 timeout 300 python tools/profile_pass.py --which 0 --batch 1 --reps 20 >> gpurun_out/pp.txt 2>&1
tail -5 gpurun_out/pp.txt
timeout 900 python -m pytest tests/test_gpu_umma.py -x -q > gpurun_out/pytest_umma.txt 2>&1
tail -30 gpurun_out/pytest_umma.txt
