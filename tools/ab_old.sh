# Same-box A/B of the current library against the round-2 baseline tree in
# _oldr2/ (a copy of commit fa3dd96 with its built library; not committed).
for c in 3 2 5 4; do
  st=40; [ $c = 5 ] && st=15
  for tree in . _oldr2; do
    (cd $tree && timeout 400 python bench.py --config $c --steps $st --warmup 5 --no-cpu-baseline --e2e-steps 1 > /tmp/ab.json 2>/dev/null)
    python -c "
import json; d=json.loads(open('/tmp/ab.json').read().strip().splitlines()[-1]); print('cfg$c', '$tree', round(d['value']), round(d['ms_per_step'],4), {k: round(v*1e3,1) for k,v in d['phases_ms_per_step'].items()})"
  done
done
