timeout 120 python tools/profile_pass.py --which 0 --batch 1 --spots 1000 --alg wgs --iters 30 --reps 50 > gpurun_out/umma_t.txt 2>&1
HS_UMMA_TRACE=1 timeout 120 python tools/profile_pass.py --which 0 --batch 1 --spots 1000 --alg wgs --iters 30 --reps 5 >> gpurun_out/umma_t.txt 2>&1
for i in 1 2; do timeout 120 python tools/profile_pass.py --which 0 --batch 32 --reps 100 >> gpurun_out/umma_t.txt 2>&1; done
HS_UMMA_TRACE=1 timeout 120 python tools/profile_pass.py --which 0 --batch 32 --reps 5 >> gpurun_out/umma_t.txt 2>&1
timeout 300 python bench.py --workload cfg4 --steps 20 --no-cpu >> gpurun_out/umma_t.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.txt 2>&1
