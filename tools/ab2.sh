# A/B of the stream-kernel variants (bench cfg3) + parity of the default path
python -m pytest tests -m gpu -x -q 2>&1 | tail -3
for v in ldg wt; do DSDE_STREAM=$v python bench.py --steps 50 --warmup 5 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ab_$v.json 2>gpurun_out/ab_$v.err; done
python - <<'PY'
import json
for v in ["ldg","wt"]:
    try:
        d = json.loads(open(f"gpurun_out/ab_{v}.json").read().strip().splitlines()[-1])
        print(v, round(d["value"]), round(d["ms_per_step"], 4), {k: round(x * 1e3, 1) for k, x in d["verify_pass"]["ms_per_step"].items()}, round(d["roofline"]["frac"], 3))
    except Exception as e:
        print(v, "failed", e)
PY
bash tools/run_variants.sh "nv4s3:-DDSDE_NV_BF16=4 -DDSDE_WT_STAGES=3" "nv4s2m3:-DDSDE_NV_BF16=4 -DDSDE_WT_STAGES=2 -DDSDE_WT_MINB=3" "nv6s2:-DDSDE_NV_BF16=6 -DDSDE_WT_STAGES=2" "nv4s4w4:-DDSDE_NV_BF16=4 -DDSDE_WT_STAGES=4 -DDSDE_WT_WARPS=4 -DDSDE_WT_MINB=4" "nv2s4m4:-DDSDE_NV_BF16=2 -DDSDE_WT_STAGES=4 -DDSDE_WT_MINB=4"
