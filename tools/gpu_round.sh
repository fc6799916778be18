# One GPU round trip: parity tests, then short benches of configs 3/4/2.
#   gpurun --timeout 1500 -- 'bash tools/gpu_round.sh TAG'
TAG=${1:-x}
mkdir -p gpurun_out/$TAG
timeout 900 python -m pytest tests -m gpu -x -q --durations=5 > gpurun_out/$TAG/gt.log 2>&1; tail -15 gpurun_out/$TAG/gt.log
for c in 3 4 2; do
  timeout 300 python bench.py --config $c --steps 40 --warmup 5 --no-cpu-baseline --e2e-steps 1 > gpurun_out/$TAG/b$c.json 2>gpurun_out/$TAG/b$c.err
  python - <<PY
import json
try:
    d = json.loads(open('gpurun_out/$TAG/b$c.json').read().strip().splitlines()[-1])
    print('cfg$c', round(d['value']), 'ms', round(d['ms_per_step'], 4), 'pass', round(d['roofline']['avg_launch_ms'], 4),
          'frac', round(d['roofline']['frac'], 3), 'whole', round(d['whole_step']['frac'], 3), d['phases_ms_per_step'])
except Exception as e:
    print('cfg$c failed', e, open('gpurun_out/$TAG/b$c.err').read()[-1500:])
PY
done
