# ncu --set full of the stream and tail kernels (one launch each, bench cfg3 shapes)
ncu --set full --clock-control none --import-source on -k regex:"k_stream_ldg|k_tail" -s 4 -c 2 \
  -o gpurun_out/prof_tail -f python bench.py --steps 3 --warmup 3 --preroll 32 --record 4 --no-cpu-baseline --e2e-steps 1 > gpurun_out/prof_tail.log 2>&1
echo ncu exit $?
python bench.py --steps 50 --warmup 5 --no-cpu-baseline --e2e-steps 1 > gpurun_out/b_nv8.json 2>gpurun_out/b_nv8.err; tail -c 600 gpurun_out/b_nv8.json
