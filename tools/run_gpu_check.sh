# GPU round trip: parity tests, bench (default path), ncu launch list + one full
# capture of the stream and tail kernels. Usage (from the repo root):
#   gpurun --timeout 1500 -- 'bash tools/run_gpu_check.sh'
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
python bench.py --steps 100 --warmup 5 --no-cpu-baseline --e2e-steps 1 > gpurun_out/bench_chk.json 2>gpurun_out/bench_chk.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_chk.csv \
  python bench.py --steps 3 --warmup 3 --preroll 2 --record 4 --no-cpu-baseline --e2e-steps 1 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_stream_ldg|k_tail" -s 6 -c 2 \
  -o gpurun_out/prof_chk -f python bench.py --steps 3 --warmup 3 --preroll 2 --record 1 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ncu_chk.log 2>&1
echo exit $?
