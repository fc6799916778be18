# parity + default bench (+ optional extra command)
python -m pytest tests -m gpu -x -q 2>&1 | tail -4
python bench.py --steps 50 --warmup 5 --no-cpu-baseline --e2e-steps 1 > gpurun_out/b_chk.json 2>gpurun_out/b_chk.err
python - <<'PY'
import json
try:
    d = json.loads(open("gpurun_out/b_chk.json").read().strip().splitlines()[-1])
    print(round(d["value"]), round(d["ms_per_step"], 4), {k: round(x * 1e3, 1) for k, x in d["verify_pass"]["ms_per_step"].items()}, round(d["roofline"]["frac"], 3))
except Exception as e:
    print("bench failed", e, open("gpurun_out/b_chk.err").read()[-1500:])
PY
