set -x
python -m pytest tests -m gpu -x -q 2>&1 | tail -3
DSDE_STREAM=tma python -m pytest tests/test_gpu_verify.py -m gpu -x -q 2>&1 | tail -3
for v in ldg tma; do DSDE_STREAM=$v python bench.py --steps 50 --warmup 5 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ab_$v.json 2>gpurun_out/ab_$v.err; done
DSDE_NVCC_FLAGS=-DDSDE_LDG_MINB=3 python paper_2509_01083_b200/_build.py --force
python bench.py --steps 50 --warmup 5 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ab_ldg3.json 2>gpurun_out/ab_ldg3.err
