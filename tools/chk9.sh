for f in "-DDSDE_NO_FAST_DRAW" "-DDSDE_FAST_MINTV=0.0" "-DDSDE_FAST_MINTV=0.0 -DDSDE_FAST_CUT=-30.f" "-DDSDE_FAST_MINTV=0.0 -DDSDE_FAST_CUT=1.f"; do
  DSDE_NVCC_FLAGS="$f" python paper_2509_01083_b200/_build.py --force > /dev/null 2>&1
  timeout 150 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --e2e-steps 1 > gpurun_out/b_x.json 2>gpurun_out/b_x.err
  python - "$f" <<'PY'
import json, sys
try:
    d = json.loads(open("gpurun_out/b_x.json").read().strip().splitlines()[-1])
    print(sys.argv[1], round(d["value"]), {k: round(x * 1e3, 1) for k, x in d["verify_pass"]["ms_per_step"].items()})
except Exception as e:
    print(sys.argv[1], "failed", e, open("gpurun_out/b_x.err").read()[-800:])
PY
done
