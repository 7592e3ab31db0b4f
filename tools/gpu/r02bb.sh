timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/r02bb_pytest.log 2>&1; tail -2 gpurun_out/r02bb_pytest.log
for tool in memcheck racecheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 5 python -m pytest tests/test_gpu_pack.py -m gpu -x -q -p no:cacheprovider \
    -k "not full_size and not 4096 and not 24 and not suite" > gpurun_out/san_${tool}_banded.txt 2>&1
  echo "$tool rc=$? $(grep -E 'passed|failed' gpurun_out/san_${tool}_banded.txt | tail -1) $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' gpurun_out/san_${tool}_banded.txt | tail -1)"
done
