: > gpurun_out/e2e_sweep.txt
for r in 1 2; do for f in 0.375 0.5 0.625; do
  echo -n "frac $f " >> gpurun_out/e2e_sweep.txt
  HS_E2E_F64_FRAC=$f timeout 300 python bench.py --steps 100 --no-cpu 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), round(d['e2e']['value']))" >> gpurun_out/e2e_sweep.txt
done; done
