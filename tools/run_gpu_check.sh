# GPU round trip: parity tests, bench (default path), ncu launch list + full capture of the top kernels
python -m pytest tests -m gpu -x -q 2>&1 | tail -3
DSDE_STREAM=tma python -m pytest tests/test_gpu_verify.py -m gpu -x -q 2>&1 | tail -2
python bench.py --steps 50 --warmup 5 --no-cpu-baseline --e2e-steps 1 > gpurun_out/bench_chk.json 2>gpurun_out/bench_chk.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 80 --csv --log-file gpurun_out/launches_chk.csv \
  python bench.py --steps 3 --warmup 3 --preroll 2 --record 4 --no-cpu-baseline --e2e-steps 1 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_stream_ldg|k_draw_ldg|k_finalize|k_select" -c 4 \
  -o gpurun_out/prof_chk -f python bench.py --steps 3 --warmup 3 --preroll 2 --record 4 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ncu_chk.log 2>&1
echo exit $?
