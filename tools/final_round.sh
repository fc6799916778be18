# Final round measurement: tools/measure_round.sh plus an ncu capture of the
# D23 path (config 4, --resample proposal).
R=${1:-m3}
bash tools/measure_round.sh $R
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_tail" -s 2 -c 1 \
  -o gpurun_out/$R/full_cfg4_d23 python bench.py --config 4 --resample proposal --steps 3 --warmup 3 --preroll 2 --record 1 --no-cpu-baseline --e2e-steps 1 > gpurun_out/$R/ncu_cfg4_d23.log 2>&1
ls -la gpurun_out/$R | tail -3
