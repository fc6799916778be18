"""Fig. SL_cap_test analogue: simulated decode
throughput for batch sizes 1..64 with and without the adaptive SL cap, the
library doing every verification step on the GPU (sim/). Writes JSON.

usage: python tools/cap_scaling.py [--out profiles/r2_cap_scaling.json] [--budget 64]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import sim  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default="profiles/r2_cap_scaling.json")
    ap.add_argument("--budget", type=int, default=64)
    ap.add_argument("--V", type=int, default=32000)
    ap.add_argument("--seeds", type=int, default=3)
    args = ap.parse_args()
    cost = sim.CostModel()
    runs = []
    for seed in range(args.seeds):
        runs.append(sim.throughput_scaling(budget=args.budget, cost=cost, V=args.V, seed=11 + seed,
                                           profiles=("code", "dialogue", "low")))
    res = {"cost_model": vars(cost), "budget": args.budget, "V": args.V,
           "profiles": ["code", "dialogue", "low"], "runs": runs}
    for name in ("cap", "no_cap"):
        res[f"mean_scaling_{name}"] = {str(r["B"]): sum(run[name][j]["scaling"] for run in runs) / len(runs)
                                       for j, r in enumerate(runs[0][name])}
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    with open(args.out, "w") as f:
        json.dump(res, f, indent=1)
    print(json.dumps({k: v for k, v in res.items() if k.startswith("mean")}))


if __name__ == "__main__":
    main()
