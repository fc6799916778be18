for f in "" "-DDSDE_FUSED_NODRAW_A" "-DDSDE_FUSED_RELAXED" "-DDSDE_FUSED_NODRAW_A -DDSDE_FUSED_RELAXED"; do
  echo "=== flags: $f"
  DSDE_NVCC_FLAGS="-DDSDE_FUSED_TRACE $f" python paper_2509_01083_b200/_build.py --force > /dev/null 2>&1
  timeout 120 python tools/trace_fused.py 2>&1 | grep -A40 "iteration 0" | grep -v iteration | sort -t' ' -k5 -n | tail -14
done
