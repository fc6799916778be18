# Round-1 vs current k_tail on the same box (measurement only; needs the
# round-1 worktree at r1wt/, `git worktree add r1wt cb4f0c8`):
# ncu --set full of one closed-loop k_tail launch of each, phase traces of
# each (trace builds), then both libraries rebuilt without the trace.
#   gpurun -- 'bash tools/experimental/ab_tail_r1.sh OUTDIR'
O=gpurun_out/$1; mkdir -p $O
R=$(pwd)
for c in 3 4; do
  (cd r1wt && timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_tail -s 40 -c 1 \
     -o $R/$O/r1_tail_c$c python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 \
     > $R/$O/r1_ncu_c$c.log 2>&1)
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_tail -s 40 -c 1 \
     -o $O/r2_tail_c$c python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 \
     > $O/r2_ncu_c$c.log 2>&1
done
(cd r1wt && DSDE_NVCC_FLAGS=-DDSDE_TAIL_TRACE=1 python paper_2509_01083_b200/_build.py --force > $R/$O/r1_build_trace.log 2>&1 \
  && for c in 3 4; do timeout 300 python tools/tail_trace.py --config $c --steps 40 > $R/$O/r1_trace_c$c.txt 2>&1; done
  python paper_2509_01083_b200/_build.py --force > /dev/null 2>&1)
DSDE_NVCC_FLAGS=-DDSDE_TAIL_TRACE=1 python paper_2509_01083_b200/_build.py --force > $O/r2_build_trace.log 2>&1 \
  && for c in 3 4; do timeout 300 python tools/tail_trace.py --config $c --steps 40 > $O/r2_trace_c$c.txt 2>&1; done
python paper_2509_01083_b200/_build.py --force > /dev/null 2>&1
for c in 3 4; do
  (cd r1wt && timeout 300 python bench.py --config $c --steps 40 --warmup 5 --no-cpu-baseline --e2e-steps 1 > $R/$O/r1_b$c.json 2>/dev/null)
  timeout 300 python bench.py --config $c --steps 40 --warmup 5 --no-cpu-baseline --e2e-steps 1 > $O/r2_b$c.json 2>/dev/null
done
ls -la $O
