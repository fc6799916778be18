# Round measurement on one B200 (gpurun): GPU tests, bench lines of every config
# (D7 default; config 4 also with the D23 recovery draw), the reference arm, the
# ncu launch list and full ncu captures of both kernels.
#   gpurun --timeout 3000 -- 'bash tools/measure_round.sh r2'
R=${1:-r2}
O=gpurun_out/$R
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/gpu.txt
timeout 1200 python -m pytest tests -m gpu -q > $O/gpu_tests.log 2>&1; tail -2 $O/gpu_tests.log
timeout 600 python bench.py > $O/bench_cfg3.json 2> $O/bench_cfg3.err
for c in 1 2 4 6; do timeout 600 python bench.py --config $c --steps 100 --warmup 10 > $O/bench_cfg$c.json 2> $O/bench_cfg$c.err; done
timeout 600 python bench.py --config 4 --steps 100 --warmup 10 --resample proposal > $O/bench_cfg4_d23.json 2> $O/bench_cfg4_d23.err
timeout 600 python bench.py --resample proposal --steps 100 --warmup 10 > $O/bench_cfg3_d23.json 2> $O/bench_cfg3_d23.err
timeout 900 python bench.py --config 5 --steps 30 --warmup 5 --cpu-seconds 10 > $O/bench_cfg5.json 2> $O/bench_cfg5.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > $O/reference.json 2> $O/reference.err
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_stream_ldg|k_tail" -c 20 --csv --log-file $O/launches_cfg3.csv \
  python bench.py --steps 6 --warmup 3 --preroll 2 --record 4 --no-cpu-baseline --e2e-steps 1 > /dev/null 2>&1
for c in 3 4; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_stream_ldg|k_tail" -s 4 -c 2 \
    -o $O/full_cfg$c python bench.py --config $c --steps 3 --warmup 3 --preroll 2 --record 1 --no-cpu-baseline --e2e-steps 1 > $O/ncu_cfg$c.log 2>&1
done
ls -la $O
