for f in "" "--no-phase-events"; do
  timeout 150 python bench.py --steps 100 --warmup 5 --no-cpu-baseline --e2e-steps 1 $f > gpurun_out/b_x.json 2>gpurun_out/b_x.err
  python - "$f" <<'PY'
import json, sys
try:
    d = json.loads(open("gpurun_out/b_x.json").read().strip().splitlines()[-1])
    print(sys.argv[1], round(d["value"]), round(d["ms_per_step"]*1e3, 1), d["verify_pass"]["event_ms_per_step"]*1e3)
except Exception as e:
    print(sys.argv[1], "failed", e, open("gpurun_out/b_x.err").read()[-600:])
PY
done
