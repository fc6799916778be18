export DSDE_BENCH_IGNORE_ERRORS=1
bash tools/run_variants.sh "base:" "pfd1:-DDSDE_PF_DRAFT=1" "pfd2:-DDSDE_PF_DRAFT=2"
