"""Per-CTA %globaltimer timeline of the last Euler step of a config-1 CIM call
(option "timeline"): when do the tile CTAs start / finish, when do the update CTAs
become resident, pass the PDL wait and exit.  Run on the B200 box.
Output: gpurun_out/timeline_<dtype>.npz + gpurun_out/timeline_summary.json."""
from __future__ import annotations

import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2405_00366_b200 as P  # noqa: E402
from paper_2405_00366_b200 import workloads as W  # noqa: E402


def q(x):
    x = np.asarray(x, float)
    return [round(float(v), 2) for v in (x.min(), np.percentile(x, 25), np.median(x),
                                         np.percentile(x, 75), x.max())]


def main():
    dts = sys.argv[1].split(",") if len(sys.argv) > 1 else ["f32"]
    insts, R, hp, _ = W.config1(0, 64)
    hp = P.baseline_params(velo=1, n_steps=300)
    B, N = len(insts), insts[0].N
    rng = np.random.default_rng(0)
    Rs = np.abs(rng.normal(size=(B, R, N))) * 0.1
    c0 = rng.normal(scale=1e-2, size=(B, R, N))
    out = {}
    for dt in dts:
        for ov in ((0, 1) if dt == "f64" else (0,)):  # fp64: item flags off / on
            with P.Context(0, dt) as ctx:
                ctx.set_option("timeline", 1)
                if dt == "f64":
                    ctx.set_option("overlap_update", ov)
                ctx.set_problems(insts)
                ctx.build_coupling()
                for _ in range(2):
                    ctx.run_cim(R, "mfz-bn", hp, 0.5, Rs, c0)
                tl = ctx.timeline().astype(np.int64)
            np.savez_compressed(os.path.join(ROOT, "gpurun_out", f"timeline_{dt}_flags{ov}.npz"), tl=tl)
            tile = tl[:256]
            tile = tile[tile[:, 0] > 0]
            upd = tl[256:8192]
            upd = upd[upd[:, 0] > 0]
            t0 = tile[:, 0].min()
            us = lambda a: (a - t0) / 1e3
            rec = {
                "tile_ctas": int(len(tile)), "update_ctas": int(len(upd)),
                "tile_entry_us": q(us(tile[:, 0])), "tile_past_wait_us": q(us(tile[:, 1])),
                "tile_last_item_us": q(us(tile[:, 2])),
                "upd_entry_us": q(us(upd[:, 0])), "upd_past_wait_us": q(us(upd[:, 1])),
                "upd_exit_us": q(us(upd[:, 2])),
                "upd_run_us": q((upd[:, 2] - upd[:, 1]) / 1e3),
                "upd_exit_after_last_tile_item_us": round(float(us(upd[:, 2]).max() - us(tile[:, 2]).max()), 2),
            }
            nrb = len(upd) // B
            fin = us(upd[:, 1]).reshape(B, nrb).min(axis=1)
            rec["instance_update_start_us_by_b"] = [round(float(v), 1) for v in fin[::4]]
            out[f"{dt}_flags{ov}"] = rec
            print(f"{dt}_flags{ov}", json.dumps(rec), flush=True)
    with open(os.path.join(ROOT, "gpurun_out", "timeline_summary.json"), "w") as f:
        json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
