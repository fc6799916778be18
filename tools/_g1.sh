bash tools/gpu_round.sh r2a
cd r1wt
for c in 3 4; do timeout 300 python bench.py --config $c --steps 40 --warmup 5 --no-cpu-baseline --e2e-steps 1 > ../gpurun_out/r2a/r1_b$c.json 2>../gpurun_out/r2a/r1_b$c.err; tail -c 700 ../gpurun_out/r2a/r1_b$c.json; echo; done
