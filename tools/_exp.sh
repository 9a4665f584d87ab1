timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
python -c "
import json;d=json.load(open('gpurun_out/bench.json'))
print(d['value'],d['ms_per_step'],d['e2e']['value'],d['latency_ms_single_hologram'],d['gpu_launches'],d['cpu_baseline']['value'],d['clocks'])"
