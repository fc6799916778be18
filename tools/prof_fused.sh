DSDE_TAIL=fused timeout 300 ncu --set full --clock-control none --import-source on -k regex:"k_fused" -s 2 -c 1 \
  -o gpurun_out/prof_fused -f python bench.py --steps 3 --warmup 3 --preroll 8 --record 4 --no-cpu-baseline --e2e-steps 1 > gpurun_out/prof_fused.log 2>&1
echo ncu exit $?
