timeout 200 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 150 python bench.py --steps 50 --warmup 5 --no-cpu-baseline --e2e-steps 1 > gpurun_out/b_t.json 2>gpurun_out/b_t.err
timeout 150 python bench.py --config 4 --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 1 > gpurun_out/b_t4.json 2>gpurun_out/b_t4.err
python - <<'PY'
import json
for v in ["t","t4"]:
    try:
        d = json.loads(open(f"gpurun_out/b_{v}.json").read().strip().splitlines()[-1])
        print(v, round(d["value"]), round(d["ms_per_step"], 4), {k: round(x * 1e3, 1) for k, x in d["verify_pass"]["ms_per_step"].items()}, round(d["roofline"]["frac"], 3), d.get("residual_fraction"))
    except Exception as e:
        print(v, "bench failed", e, open(f"gpurun_out/b_{v}.err").read()[-1500:])
PY
