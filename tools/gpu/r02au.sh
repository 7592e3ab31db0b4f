for tool in memcheck racecheck synccheck; do
  t=test_gpu_parity
  timeout 1500 compute-sanitizer --tool $tool --print-limit 5 python -m pytest tests/$t.py -m gpu -x -q -p no:cacheprovider \
    -k "not full_size and not big and not 4096 and not 24 and not exhaustive" > gpurun_out/san_${tool}_$t.txt 2>&1
  echo "$tool $t rc=$? $(grep -E 'passed|failed' gpurun_out/san_${tool}_$t.txt | tail -1) $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' gpurun_out/san_${tool}_$t.txt | tail -1)"
done
