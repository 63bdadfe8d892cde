mkdir -p gpurun_out
CASES=${CASES:-"persist persist_fc rows tc_level fp32 ksplit_bwd multicast rows_pair dag ablations"}
python tools/sanitize_cases.py $CASES > gpurun_out/san_plain.log 2>&1; echo plain rc=$?; cat gpurun_out/san_plain.log
for tool in memcheck racecheck synccheck; do
  for c in $CASES; do
    timeout 600 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_cases.py $c > gpurun_out/san_${tool}_${c}.log 2>&1
    echo "$tool $c rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' gpurun_out/san_${tool}_${c}.log | tail -1)"
  done
done
