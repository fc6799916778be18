timeout 700 python -m pytest tests -m gpu -x -q > gpurun_out/gt.log 2>&1; tail -2 gpurun_out/gt.log
for c in 3 4 2; do timeout 200 python bench.py --config $c --steps 60 --warmup 5 --no-cpu-baseline --e2e-steps 1 > gpurun_out/b$c.json 2>/dev/null; python -c "
import json; d=json.loads(open('gpurun_out/b$c.json').read().strip().splitlines()[-1]); print('cfg$c', round(d['value']), round(d['ms_per_step'],4), {k: round(v*1e3,1) for k,v in d['verify_pass']['ms_per_step'].items()})"; done
DSDE_NVCC_FLAGS=-DDSDE_TAIL_TRACE=1 python paper_2509_01083_b200/_build.py --force > /dev/null && timeout 300 python tools/tail_trace.py --config 2 | tail -4 && timeout 300 python tools/tail_trace.py --config 3 | tail -4
