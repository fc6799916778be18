DSDE_TAIL=fused timeout 200 python -m pytest tests/test_gpu_verify.py tests/test_gpu_signal.py -m gpu -x -q 2>&1 | tail -2
for v in fused tail; do DSDE_TAIL=$v timeout 150 python bench.py --steps 50 --warmup 5 --no-cpu-baseline --e2e-steps 1 > gpurun_out/b_$v.json 2>gpurun_out/b_$v.err; done
python - <<'PY'
import json
for v in ["fused","tail"]:
    try:
        d = json.loads(open(f"gpurun_out/b_{v}.json").read().strip().splitlines()[-1])
        print(v, round(d["value"]), round(d["ms_per_step"], 4), {k: round(x * 1e3, 1) for k, x in d["verify_pass"]["ms_per_step"].items()}, round(d["roofline"]["frac"], 3))
    except Exception as e:
        print(v, "bench failed", e, open(f"gpurun_out/b_{v}.err").read()[-1500:])
PY
