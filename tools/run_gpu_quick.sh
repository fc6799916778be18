python -m pytest tests -m gpu -x -q 2>&1 | tail -3
DSDE_STREAM=tma python -m pytest tests/test_gpu_verify.py -m gpu -x -q 2>&1 | tail -2
python bench.py --steps 50 --warmup 5 --no-cpu-baseline --e2e-steps 1 > gpurun_out/bench_q.json 2>gpurun_out/bench_q.err
python - <<'PY'
import json
d = json.loads(open("gpurun_out/bench_q.json").read().strip().splitlines()[-1])
print(round(d["value"]), round(d["ms_per_step"], 4), {k: round(x * 1e3, 1) for k, x in d["verify_pass"]["ms_per_step"].items()}, round(d["roofline"]["frac"], 3))
PY
