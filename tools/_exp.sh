mkdir -p gpurun_out/san
timeout 900 compute-sanitizer --tool racecheck --print-limit 5 python tools/sanitize.py > gpurun_out/san/racecheck_f16.txt 2>&1; echo "rc=$?" >> gpurun_out/san/racecheck_f16.txt
HS_LIB_PATH=abtest/tf32.so timeout 900 compute-sanitizer --tool racecheck --print-limit 5 python tools/sanitize.py > gpurun_out/san/racecheck_tf32.txt 2>&1; echo "rc=$?" >> gpurun_out/san/racecheck_tf32.txt
