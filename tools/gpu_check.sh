mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "cfg5" > gpurun_out/pytest_cfg5.log 2>&1; echo cfg5 rc=$?; tail -3 gpurun_out/pytest_cfg5.log
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo gpu rc=$?; tail -5 gpurun_out/pytest_gpu.log
python tools/sanitize_cases.py > gpurun_out/san_plain.log 2>&1; echo plain rc=$?; cat gpurun_out/san_plain.log
for tool in memcheck racecheck synccheck; do
  for c in persist persist_fc rows tc_level fp32; do
    timeout 600 compute-sanitizer --tool $tool --print-limit 50 python tools/sanitize_cases.py $c > gpurun_out/san_${tool}_${c}.log 2>&1
    echo "$tool $c rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' gpurun_out/san_${tool}_${c}.log | tail -1)"
  done
done
