"""fp64 DMMA path: item flags (option overlap_update) off / on at BASELINE config 1 --
time per Euler step, refit time, and that the results are bitwise equal (only WHEN an
update CTA runs changes).  Run on the B200 box.  Output: gpurun_out/overlap64.json"""
from __future__ import annotations
import json, os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2405_00366_b200 as P  # noqa: E402
from paper_2405_00366_b200 import workloads as W  # noqa: E402


def main():
    alts = int(sys.argv[1]) if len(sys.argv) > 1 else 2
    insts, R, hp, _ = W.config1(0, 64)
    hp = P.baseline_params(velo=alts - 1, n_steps=hp.n_steps)
    seeds = P.replica_seeds(insts, R, "mfz-bn")
    out, ref = {"alts": alts, "n_steps": hp.n_steps}, None
    for ov in (0, 1):
        with P.Context(0, "f64") as ctx:
            ctx.set_option("overlap_update", ov)
            ctx.set_problems(insts)
            ctx.build_coupling()
            best = None
            for _ in range(2):
                res = ctx.solve(R, "mfz-bn", hp, seeds)
                tm = ctx.timing()
                if best is None or tm["cim_ms"] < best["cim_ms"]:
                    best = dict(tm)
        rec = {"step_us": 1e3 * best["cim_ms"] / (alts * hp.n_steps), "refit_ms": best["refit_ms"],
               "total_ms": best["total_ms"]}
        if ref is None:
            ref = res
        else:
            rec["bitwise_equal_to_no_overlap"] = bool(
                np.array_equal(ref["R"], res["R"]) and np.array_equal(ref["sigma"], res["sigma"]))
        out[f"overlap{ov}"] = rec
        print(f"f64 overlap{ov}", json.dumps(rec), flush=True)
    json.dump(out, open(os.path.join(ROOT, "gpurun_out", "overlap64.json"), "w"), indent=1)


if __name__ == "__main__":
    main()
