./tools/pipe_bench 2>&1 | tail -12
bash tools/run_variants.sh "ldg_nv4m4:-DDSDE_NV_BF16=4 -DDSDE_LDG_MINB=4" "ldg_nv6m4:-DDSDE_LDG_MINB=4" "ldg_nv3m5:-DDSDE_NV_BF16=3 -DDSDE_LDG_MINB=5" "ldg_nv8m3:-DDSDE_NV_BF16=8 -DDSDE_LDG_MINB=3" "ldg_exp2:-DDSDE_EXPERIMENT=2" "ldg_exp1:-DDSDE_EXPERIMENT=1"
