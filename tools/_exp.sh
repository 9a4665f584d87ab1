# scratch driver for one gpurun experiment (the last one run is kept here)
mkdir -p gpurun_out/r2
rm -f gpurun_out/e2e_sweep.txt
for c in 4 8 16; do for f in 0.25 0.375; do
  echo "chunks $c frac $f" >> gpurun_out/e2e_sweep.txt
  HS_WIDEN_CHUNKS=$c HS_E2E_F64_FRAC=$f timeout 300 python tools/e2e_probe.py --steps 20 2>&1 | grep -E "phase=True|widening 33" >> gpurun_out/e2e_sweep.txt
done; done
timeout 600 python -m pytest tests/test_gpu_parity.py -q -k pipelined > gpurun_out/pipe_test.txt 2>&1
