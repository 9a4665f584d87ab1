mkdir -p gpurun_out
for u in 1 0; do HS_UMMA=$u timeout 600 python tools/_n600.py 2>&1 | grep max; done
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.txt 2>&1
tail -3 gpurun_out/pytest_gpu.txt
