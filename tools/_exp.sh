timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.txt 2>&1
tail -3 gpurun_out/pytest_gpu.txt
for r in 1 2; do timeout 600 python bench.py --no-cpu > gpurun_out/bench.json 2> gpurun_out/bench.err
python -c "
import json;d=json.load(open('gpurun_out/bench.json'))
print(d['value'],d['ms_per_step'],d['e2e']['value'],d['latency_ms_single_hologram'],d['gpu_launches'])"; done
