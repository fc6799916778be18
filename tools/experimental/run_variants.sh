# Build-flag A/B of the streaming kernels on the GPU box: one bench line per variant.
# usage: bash tools/run_variants.sh "name1:flags1" "name2:flags2" ...
for spec in "$@"; do
  name="${spec%%:*}"; flags="${spec#*:}"
  DSDE_NVCC_FLAGS="$flags" python paper_2509_01083_b200/_build.py --force > /dev/null 2>&1 || { echo "$name build failed"; continue; }
  python bench.py --steps 50 --warmup 5 --no-cpu-baseline --e2e-steps 1 > gpurun_out/var_$name.json 2> gpurun_out/var_$name.err
  python - "$name" <<'PY'
import json, sys
n = sys.argv[1]
try:
    d = json.loads(open(f"gpurun_out/var_{n}.json").read().strip().splitlines()[-1])
    print(n, round(d["value"]), round(d["ms_per_step"], 4), {k: round(x * 1e3, 1) for k, x in d["verify_pass"]["ms_per_step"].items()}, round(d["roofline"]["frac"], 3))
except Exception as e:
    print(n, "failed", e)
PY
done
