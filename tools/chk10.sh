timeout 200 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for c in 3 2 4; do timeout 150 python bench.py --config $c --steps 30 --warmup 5 --no-cpu-baseline --e2e-steps 1 > gpurun_out/b_c$c.json 2>gpurun_out/b_c$c.err; done
DSDE_STREAM=tma timeout 150 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/b_tma.json 2>gpurun_out/b_tma.err
python - <<'PY'
import json
for v in ["c3","c2","c4","tma"]:
    try:
        d = json.loads(open(f"gpurun_out/b_{v}.json").read().strip().splitlines()[-1])
        print(v, round(d["value"]), round(d["ms_per_step"], 4), {k: round(x * 1e3, 1) for k, x in d["verify_pass"]["ms_per_step"].items()}, round(d["roofline"]["frac"], 3))
    except Exception as e:
        print(v, "bench failed", e, open(f"gpurun_out/b_{v}.err").read()[-1500:])
PY
