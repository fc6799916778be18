timeout 200 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for f in "" "-DDSDE_TAIL_CPA=0"; do
DSDE_NVCC_FLAGS="$f" python paper_2509_01083_b200/_build.py --force > /dev/null 2>&1
for c in 3 4 2; do
  timeout 150 python bench.py --config $c --steps 40 --warmup 5 --no-cpu-baseline --e2e-steps 1 > gpurun_out/b_x.json 2>gpurun_out/b_x.err
  python - "$f cfg$c" <<'PY'
import json, sys
try:
    d = json.loads(open("gpurun_out/b_x.json").read().strip().splitlines()[-1])
    print(sys.argv[1], round(d["value"]), {k: round(x * 1e3, 1) for k, x in d["verify_pass"]["ms_per_step"].items()}, round(d["roofline"]["frac"], 3))
except Exception as e:
    print(sys.argv[1], "failed", e, open("gpurun_out/b_x.err").read()[-600:])
PY
done; done
