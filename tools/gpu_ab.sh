# A/B of the recovery-draw readings on one box: bench configs 3/4/2 with the
# D23 default and with --resample full.
#   gpurun --timeout 1500 -- 'bash tools/gpu_ab.sh TAG'
TAG=${1:-x}
mkdir -p gpurun_out/$TAG
for c in 3 4 2; do
  for rs in proposal full; do
    timeout 300 python bench.py --config $c --steps 40 --warmup 5 --no-cpu-baseline --e2e-steps 1 --resample $rs > gpurun_out/$TAG/b$c$rs.json 2>gpurun_out/$TAG/b$c$rs.err
    python - <<PY
import json
try:
    d = json.loads(open('gpurun_out/$TAG/b$c$rs.json').read().strip().splitlines()[-1])
    print('cfg$c $rs', round(d['value']), 'ms', round(d['ms_per_step'], 4), 'stream', round(d['roofline']['avg_launch_ms'], 4),
          'frac', round(d['roofline']['frac'], 3), 'whole', round(d['whole_step']['frac'], 3), d['phases_ms_per_step'], d['parity'])
except Exception as e:
    print('cfg$c $rs failed', e, open('gpurun_out/$TAG/b$c$rs.err').read()[-1500:])
PY
  done
done
