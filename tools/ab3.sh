# parity (fused tail + dsde_step) then stream-variant A/B incl. wt2
python -m pytest tests -m gpu -x -q 2>&1 | tail -4
for v in ldg wt2; do DSDE_STREAM=$v python bench.py --steps 50 --warmup 5 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ab_$v.json 2>gpurun_out/ab_$v.err; done
DSDE_TAIL=split python bench.py --steps 50 --warmup 5 --no-cpu-baseline --e2e-steps 1 --split-calls > gpurun_out/ab_split.json 2>gpurun_out/ab_split.err
python - <<'PY'
import json
for v in ["ldg","wt2","split"]:
    try:
        d = json.loads(open(f"gpurun_out/ab_{v}.json").read().strip().splitlines()[-1])
        print(v, round(d["value"]), round(d["ms_per_step"], 4), {k: round(x * 1e3, 1) for k, x in d["verify_pass"]["ms_per_step"].items()}, round(d["roofline"]["frac"], 3))
    except Exception as e:
        print(v, "failed", e, open(f"gpurun_out/ab_{v}.err").read()[-800:])
PY
export DSDE_STREAM=wt2
bash tools/run_variants.sh "w2nv4s3:-DDSDE_NV_BF16=4 -DDSDE_W2_STAGES=3" "w2nv6s2:-DDSDE_W2_STAGES=2" "w2nv8s2:-DDSDE_NV_BF16=8 -DDSDE_W2_STAGES=2" "w2nv8s3w2:-DDSDE_NV_BF16=8 -DDSDE_W2_STAGES=3 -DDSDE_W2_WARPS=2 -DDSDE_W2_MINB=4" "w2nv4s4w2:-DDSDE_NV_BF16=4 -DDSDE_W2_STAGES=4 -DDSDE_W2_WARPS=2 -DDSDE_W2_MINB=6"
