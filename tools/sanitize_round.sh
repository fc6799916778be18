# compute-sanitizer over a representative subset of the GPU tests (gpurun).
R=${1:-r2}
O=gpurun_out/$R
mkdir -p $O
for tool in memcheck racecheck synccheck initcheck; do
  echo "== $tool" >> $O/sanitizer.txt
  timeout 1500 compute-sanitizer --tool $tool --error-exitcode 7 --print-limit 20 \
    python -m pytest -q -x -m gpu "tests/test_gpu_verify.py::test_verify_parity" tests/test_gpu_vocab.py \
    "tests/test_gpu_temp_mask.py::test_masked_parity" "tests/test_gpu_signal.py::test_step_matches_three_calls" \
    tests/test_gpu_entropy.py >> $O/sanitizer.txt 2>&1
  echo "exit $?" >> $O/sanitizer.txt
done
grep -E "^== |ERROR SUMMARY|^exit|passed|failed" $O/sanitizer.txt
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_stream|k_tail" -c 40 --csv --log-file $O/launches_ours_cfg3.csv \
  python bench.py --steps 6 --warmup 3 --preroll 2 --record 4 --no-cpu-baseline --e2e-steps 1 > /dev/null 2>&1
tail -3 $O/launches_ours_cfg3.csv
