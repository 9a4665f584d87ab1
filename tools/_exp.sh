mkdir -p gpurun_out
for w in 0 2; do timeout 300 python tools/profile_pass.py --which $w --batch 32 --reps 20; done
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.txt 2>&1
tail -3 gpurun_out/pytest_gpu.txt
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
python -c "
import json;d=json.load(open('gpurun_out/bench.json'))
print(d['value'],d['ms_per_step'],d['e2e']['value'],d['latency_ms_single_hologram'],d['roofline']['full_pass']['ms_per_launch'],d['roofline']['ms_per_launch'])"
