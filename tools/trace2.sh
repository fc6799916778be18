# Measurement build with DSDE_TAIL_TRACE=2 (phase stamps + a repeated select),
# D7 traces of configs 3/4, then the product build and D7 benches.
DSDE_NVCC_FLAGS=-DDSDE_TAIL_TRACE=2 python paper_2509_01083_b200/_build.py --force > /dev/null || exit 1
for c in 3 4; do timeout 300 python tools/tail_trace.py --config $c --resample 1 | tail -3; done
python paper_2509_01083_b200/_build.py --force > /dev/null
for c in 3 4 2; do
  timeout 300 python bench.py --config $c --steps 40 --warmup 5 --no-cpu-baseline --e2e-steps 1 > gpurun_out/t2_b$c.json 2>/dev/null
  python -c "
import json; d=json.loads(open('gpurun_out/t2_b$c.json').read().strip().splitlines()[-1]); print('cfg$c', round(d['value']), round(d['ms_per_step'],4), d['phases_ms_per_step'])"
done
