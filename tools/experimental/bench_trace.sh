# bench configs $CFGS (default "3 4") with the in-tree library, then a k_tail
# phase trace of each (trace build), then the normal build again.
#   gpurun -- 'bash tools/experimental/bench_trace.sh OUTDIR'
O=gpurun_out/$1; mkdir -p $O
for c in ${CFGS:-3 4}; do
  timeout 300 python bench.py --config $c --steps 40 --warmup 5 --no-cpu-baseline --e2e-steps 1 > $O/b$c.json 2>$O/b$c.err
  python -c "
import json
d=json.loads(open('$O/b$c.json').read().strip().splitlines()[-1])
print('cfg$c', round(d['value']), 'ms', round(d['ms_per_step'],4), 'stream', round(d['roofline']['avg_launch_ms'],4), 'frac', round(d['roofline']['frac'],3), 'whole', round(d['whole_step']['frac'],3), 'parity', d.get('parity'))" 2>&1 | tail -1
done
if [ -z "$NOTRACE" ]; then
DSDE_NVCC_FLAGS=-DDSDE_TAIL_TRACE=1 python paper_2509_01083_b200/_build.py --force > $O/build_trace.log 2>&1 \
  && for c in ${CFGS:-3 4}; do timeout 300 python tools/tail_trace.py --config $c --steps 40 > $O/trace_c$c.txt 2>&1; cat $O/trace_c$c.txt; done
python paper_2509_01083_b200/_build.py --force > /dev/null 2>&1
fi
