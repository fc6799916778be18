set -x
for v in ldg tma; do DSDE_STREAM=$v python bench.py --steps 50 --warmup 5 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ab_$v.json 2>gpurun_out/ab_$v.err; done
bash tools/run_variants.sh "pf2:-DDSDE_LDG_PREFETCH=1 -DDSDE_LDG_MINB=2" "nv4:-DDSDE_NV_BF16=4" "nv4pf:-DDSDE_NV_BF16=4 -DDSDE_LDG_PREFETCH=1" "nv3pf:-DDSDE_NV_BF16=3 -DDSDE_LDG_PREFETCH=1 -DDSDE_LDG_MINB=4" "exp1:-DDSDE_EXPERIMENT=1" "exp2:-DDSDE_EXPERIMENT=2"
python - <<'PY'
import json
for v in ["ldg","tma"]:
    d = json.loads(open(f"gpurun_out/ab_{v}.json").read().strip().splitlines()[-1])
    print(v, round(d["value"]), round(d["ms_per_step"], 4), {k: round(x * 1e3, 1) for k, x in d["verify_pass"]["ms_per_step"].items()}, round(d["roofline"]["frac"], 3))
PY
