rm -f gpurun_out/ring.txt
timeout 300 python tools/ab_time.py >> gpurun_out/ring.txt 2>&1
HS_UMMA_TRACE=1 timeout 300 python tools/profile_pass.py --which 0 --batch 32 >> gpurun_out/ring.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_umma.py tests/test_gpu_parity.py tests/test_gpu_spot_chunks.py -q -x > gpurun_out/ring_tests.txt 2>&1
