# One ncu --set full capture (with source counters) of k_tail at config 3.
#   gpurun --timeout 900 -- 'bash tools/ncu_tail.sh TAG'
TAG=${1:-x}
mkdir -p gpurun_out/$TAG
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_tail" -s 6 -c 1 \
  -o gpurun_out/$TAG/tail python bench.py --config ${2:-3} --steps 3 --warmup 3 --preroll 2 --record 1 --no-cpu-baseline --e2e-steps 1 > gpurun_out/$TAG/ncu.log 2>&1
ls -la gpurun_out/$TAG
