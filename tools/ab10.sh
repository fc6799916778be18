export DSDE_BENCH_IGNORE_ERRORS=1
bash tools/run_variants.sh "nvd2:-DDSDE_NVD_BF16=2" "nvd3:-DDSDE_NVD_BF16=3" "nvd6:-DDSDE_NVD_BF16=6" "nvd8:-DDSDE_NVD_BF16=8"
