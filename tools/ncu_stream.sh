# ncu --set full capture of the streaming kernels (one launch each) for source-level stall analysis
python paper_2509_01083_b200/_build.py --force > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_stream_ldg|k_draw_ldg" -s 40 -c 2 \
  -o gpurun_out/prof_${1:-cur} -f python bench.py --steps 3 --warmup 3 --preroll 32 --record 4 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ncu_${1:-cur}.log 2>&1
echo exit $?
