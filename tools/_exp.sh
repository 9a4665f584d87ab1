# scratch driver for one gpurun experiment (the last one run is kept here)
./tools/atan2_dev
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.txt 2>&1
tail -2 gpurun_out/pytest_gpu.txt
