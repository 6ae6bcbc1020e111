"""Is the symmetric tile stream bound by HBM or by what one SM keeps in flight?
Config 1, fp32 / fp64, the item schedule placed on fewer persistent CTAs
(option sched_ctas): per-step time vs CTAs.  Run on the B200 box."""
from __future__ import annotations

import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2405_00366_b200 as P  # noqa: E402
from paper_2405_00366_b200 import workloads as W  # noqa: E402


def main():
    dts = sys.argv[1].split(",") if len(sys.argv) > 1 else ["f32"]
    insts, R, hp, _ = W.config1(0, 64)
    hp = P.baseline_params(velo=1, n_steps=500)
    seeds = P.replica_seeds(insts, R, "mfz-bn")
    out = {}
    for dt in dts:
        for n in [int(x) for x in os.environ.get("CTAS", "148,132,111,96,74").split(",")]:
            with P.Context(0, dt) as ctx:
                ctx.set_option("sched_ctas", n)
                ctx.set_option("kernel_timing", 0)
                ctx.set_problems(insts)
                ctx.build_coupling()
                best = 1e9
                for _ in range(2):
                    ctx.solve(R, "mfz-bn", hp, seeds)
                    best = min(best, ctx.timing()["cim_ms"])
            out[f"{dt}_{n}"] = 1e3 * best / (2 * hp.n_steps)
            print(dt, n, "CTAs: step", round(out[f"{dt}_{n}"], 2), "us", flush=True)
    with open(os.path.join(ROOT, "gpurun_out", "cta_sweep.json"), "w") as f:
        json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
