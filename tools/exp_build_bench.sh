# Kernel experiments on the GPU box: for each "TAG:NVCC_FLAGS" argument, rebuild
# libdsde.so with those flags and bench configs $CFGS (default "3 4").
#   gpurun -- 'bash tools/exp_build_bench.sh OUTDIR "base:" "lag4:-DDSDE_PASS_LAG_ITERS=4"'
OUT=$1; shift
mkdir -p gpurun_out/$OUT
for spec in "$@"; do
  tag=${spec%%:*}; flags=${spec#*:}
  DSDE_NVCC_FLAGS="$flags" python paper_2509_01083_b200/_build.py --force > gpurun_out/$OUT/build_$tag.log 2>&1 || { echo "$tag build failed"; continue; }
  for c in ${CFGS:-3 4}; do
    timeout 300 python bench.py --config $c --steps ${STEPS:-40} --warmup 5 --no-cpu-baseline --e2e-steps 1 > gpurun_out/$OUT/${tag}_b$c.json 2>gpurun_out/$OUT/${tag}_b$c.err
    python - <<PY
import json
try:
    d = json.loads(open('gpurun_out/$OUT/${tag}_b$c.json').read().strip().splitlines()[-1])
    print('$tag cfg$c', round(d['value']), 'ms', round(d['ms_per_step'], 4), 'pass', round(d['roofline']['avg_launch_ms'], 4),
          'frac', round(d['roofline']['frac'], 3), 'whole', round(d['whole_step']['frac'], 3))
except Exception as e:
    print('$tag cfg$c failed', e, open('gpurun_out/$OUT/${tag}_b$c.err').read()[-800:])
PY
  done
done
