# Round artifacts: bench (N=1, defaults), reference arm, ncu launch list, ncu --set full
# of the stream and tail kernels (one launch each, the replayed recorded step).
set -x
python bench.py > gpurun_out/bench_r1.json 2> gpurun_out/bench_r1.err
python bench.py --impl reference --steps 10 --warmup 3 > gpurun_out/bench_ref_r1.json 2> gpurun_out/bench_ref_r1.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r1.csv \
  python bench.py --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/launches_r1.bench.json 2>&1
# full capture: preroll 2 + record 1 launches skipped -> the first warm-up step (= the recorded step)
python bench.py --steps 3 --warmup 3 --preroll 2 --record 1 --no-cpu-baseline --e2e-steps 1 > gpurun_out/full_r1.bench.json 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_stream_ldg" -s 3 -c 1 \
  -o gpurun_out/full_stream_r1 -f python bench.py --steps 3 --warmup 3 --preroll 2 --record 1 --no-cpu-baseline --e2e-steps 1 > gpurun_out/full_stream_r1.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_tail" -s 3 -c 1 \
  -o gpurun_out/full_tail_r1 -f python bench.py --steps 3 --warmup 3 --preroll 2 --record 1 --no-cpu-baseline --e2e-steps 1 > gpurun_out/full_tail_r1.log 2>&1
echo done
python bench.py --config 4 --steps 100 --warmup 5 --e2e-steps 1 --cpu-seconds 5 > gpurun_out/bench_cfg4_r1.json 2> gpurun_out/bench_cfg4_r1.err
python bench.py --config 2 --steps 200 --warmup 10 --e2e-steps 2 --cpu-seconds 5 > gpurun_out/bench_cfg2_r1.json 2> gpurun_out/bench_cfg2_r1.err
python bench.py --greedy --steps 100 --warmup 5 --e2e-steps 1 --cpu-seconds 5 > gpurun_out/bench_greedy_r1.json 2> gpurun_out/bench_greedy_r1.err
echo extra done
