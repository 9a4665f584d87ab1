L=paper_2003_05293_b200/_lib
: > gpurun_out/ab.txt
for r in 1 2 3; do
  for v in old new; do
    cp $L/$v.so.bin $L/libholospots_b200.so
    echo -n "$v " >> gpurun_out/ab.txt
    timeout 120 python tools/profile_pass.py --which 1 --batch 32 --reps 100 2>&1 | tail -1 >> gpurun_out/ab.txt
  done
done
for v in old new; do cp $L/$v.so.bin $L/libholospots_b200.so; echo -n "$v bench " >> gpurun_out/ab.txt; timeout 300 python bench.py --steps 100 --no-cpu 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), round(d['e2e']['value']), d['latency_ms_single_hologram'])" >> gpurun_out/ab.txt; timeout 120 python tools/b1_probe.py >> gpurun_out/ab.txt 2>&1; done
cp $L/new.so.bin $L/libholospots_b200.so
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.txt 2>&1
