# k_tail phase traces of build variants on one box: for each "TAG:NVCC_FLAGS",
# a trace build and tools/tail_trace.py on configs $CFGS, then a normal build
# of the same flags and a bench of each config.
#   gpurun -- 'bash tools/experimental/trace_variants.sh OUTDIR "base:" "dyn:-DDSDE_DRAW_DYN=1"'
O=gpurun_out/$1; shift; mkdir -p $O
for spec in "$@"; do
  tag=${spec%%:*}; flags=${spec#*:}
  DSDE_NVCC_FLAGS="$flags -DDSDE_TAIL_TRACE=1" python paper_2509_01083_b200/_build.py --force > $O/build_tr_$tag.log 2>&1 || { echo "$tag trace build failed"; continue; }
  for c in ${CFGS:-3 4}; do
    echo "== $tag cfg$c"; timeout 300 python tools/tail_trace.py --config $c --steps 40 2>&1 | tail -3
  done
  DSDE_NVCC_FLAGS="$flags" python paper_2509_01083_b200/_build.py --force > $O/build_$tag.log 2>&1 || continue
  for c in ${CFGS:-3 4}; do
    timeout 300 python bench.py --config $c --steps 40 --warmup 5 --no-cpu-baseline --e2e-steps 1 > $O/${tag}_b$c.json 2>/dev/null
    python -c "
import json
d=json.loads(open('$O/${tag}_b$c.json').read().strip().splitlines()[-1])
print('$tag cfg$c', round(d['value']), 'ms', round(d['ms_per_step'],4), 'stream', round(d['roofline']['avg_launch_ms'],4), 'whole', round(d['whole_step']['frac'],3))" 2>&1 | tail -1
  done
done
