# scratch driver for one gpurun experiment (the last one run is kept here)
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
python -c "
import json;d=json.load(open('gpurun_out/bench.json'))
print(d['value'],d['ms_per_step'],d['e2e']['value'],d['latency_ms_single_hologram'],d['roofline']['full_pass']['ms_per_launch'],d['roofline']['full_pass']['final_pass_ms_per_launch'],d['roofline']['frac'],d['roofline']['full_pass']['tensor']['frac'])"
