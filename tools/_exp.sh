timeout 300 python tools/b1_probe.py > gpurun_out/b1.txt 2>&1
timeout 300 python tools/b1_probe.py >> gpurun_out/b1.txt 2>&1
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.txt 2>&1
timeout 300 python bench.py > gpurun_out/bench.txt 2>&1
