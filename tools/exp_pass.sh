# Kernel experiments: for each "TAG:NVCC_FLAGS", rebuild and time tools/pass_bench.py on configs $CFGS.
OUT=$1; shift
mkdir -p gpurun_out/$OUT
for spec in "$@"; do
  tag=${spec%%:*}; flags=${spec#*:}
  DSDE_NVCC_FLAGS="$flags" python paper_2509_01083_b200/_build.py --force > gpurun_out/$OUT/build_$tag.log 2>&1 || { echo "$tag build failed"; continue; }
  for c in ${CFGS:-3}; do
    echo -n "$tag "; timeout 200 python tools/pass_bench.py --config $c 2>&1 | tail -1
  done
done
