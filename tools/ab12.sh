timeout 200 python -m pytest tests/test_gpu_verify.py tests/test_gpu_signal.py -m gpu -x -q 2>&1 | tail -2
for p in 1 0; do for c in 3 2; do
  DSDE_PDL=$p timeout 150 python bench.py --config $c --steps 100 --warmup 5 --no-cpu-baseline --e2e-steps 1 > gpurun_out/b_x.json 2>gpurun_out/b_x.err
  python - "pdl=$p cfg$c" <<'PY'
import json, sys
try:
    d = json.loads(open("gpurun_out/b_x.json").read().strip().splitlines()[-1])
    print(sys.argv[1], round(d["value"]), round(d["ms_per_step"]*1e3, 1), {k: round(x * 1e3, 1) for k, x in d["verify_pass"]["ms_per_step"].items()}, round(d["roofline"]["frac"], 3))
except Exception as e:
    print(sys.argv[1], "failed", e, open("gpurun_out/b_x.err").read()[-600:])
PY
done; done
