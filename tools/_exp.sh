timeout 900 python -m pytest tests/test_gpu_sharded.py -q > gpurun_out/sharded.txt 2>&1
timeout 400 python bench.py --gpus 2 --workload cfg4 --steps 10 --no-cpu > gpurun_out/bench_g2_cfg4.json 2> gpurun_out/bench_g2_cfg4.err
