# k_tail phase traces of both recovery-draw readings (measurement build).
#   gpurun --timeout 900 -- 'bash tools/trace_ab.sh'
DSDE_NVCC_FLAGS=-DDSDE_TAIL_TRACE=1 python paper_2509_01083_b200/_build.py --force > /dev/null || exit 1
for c in 3 4; do for rs in 0 1; do echo "resample=$rs"; timeout 300 python tools/tail_trace.py --config $c --resample $rs | tail -5; done; done
python paper_2509_01083_b200/_build.py --force > /dev/null
