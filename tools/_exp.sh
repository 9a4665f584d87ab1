timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
python -c "
import json;d=json.load(open('gpurun_out/bench.json'))
print(d['value'],d['ms_per_step'],d['e2e']['value'],d['latency_ms_single_hologram'],d['roofline']['full_pass']['ms_per_launch'],d['roofline']['full_pass']['final_pass_ms_per_launch'],d['roofline']['ms_per_launch'])"
timeout 900 python tools/bench_configs.py --out gpurun_out/configs.jsonl > gpurun_out/configs.log 2>&1
python3 -c "
import json
for l in open('gpurun_out/configs.jsonl'):
    d=json.loads(l); print(d['config'][:40], round(d['ms_per_hologram'],4), round(d['holograms_per_s'],1))
"
