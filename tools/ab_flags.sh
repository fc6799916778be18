# Same-box A/B of the product build against a build with extra nvcc flags.
#   gpurun -- 'BENCH_ARGS="--resample proposal" bash tools/ab_flags.sh "-DFOO=1" "3 2 4"'
FLAGS=$1; CFGS=${2:-"3 2 4"}
run() {
  for c in $CFGS; do
    timeout 400 python bench.py --config $c --steps 40 --warmup 5 --no-cpu-baseline --e2e-steps 1 $BENCH_ARGS > /tmp/ab.json 2>/dev/null
    python -c "
import json; d=json.loads(open('/tmp/ab.json').read().strip().splitlines()[-1]); print('cfg$c', '$1', round(d['value']), round(d['ms_per_step'],4), {k: round(v*1e3,1) for k,v in d['phases_ms_per_step'].items()})"
  done
}
run base
DSDE_NVCC_FLAGS="$FLAGS" python paper_2509_01083_b200/_build.py --force > /dev/null || exit 1
run variant
python paper_2509_01083_b200/_build.py --force > /dev/null
run base
