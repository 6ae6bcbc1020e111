"""Is the spread of the tile CTAs' finish times a property of the SM?  Config 1, fp32:
per-CTA (SM id, tiles, time from the PDL wait to the last item) of the last Euler step
of several CIM calls; correlation of the per-tile time across calls and by SM id.
Run on the B200 box.  Output: gpurun_out/sm_speed.json"""
from __future__ import annotations
import json, os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2405_00366_b200 as P  # noqa: E402
from paper_2405_00366_b200 import workloads as W  # noqa: E402

insts, R, hp, _ = W.config1(0, 64)
hp = P.baseline_params(velo=1, n_steps=200)
B, N = len(insts), insts[0].N
rng = np.random.default_rng(0)
Rs = np.abs(rng.normal(size=(B, R, N))) * 0.1
c0 = rng.normal(scale=1e-2, size=(B, R, N))
runs = []
with P.Context(0, "f32") as ctx:
    ctx.set_option("timeline", 1)
    ctx.set_problems(insts)
    ctx.build_coupling()
    for k in range(5):
        ctx.run_cim(R, "mfz-bn", hp, 0.5, Rs, c0)
        tl = ctx.timeline()
        t = tl[:148].astype(np.int64)
        smid = (tl[:148, 3] >> np.uint64(32)).astype(np.int64)
        tiles = (tl[:148, 3] & np.uint64(0xffffffff)).astype(np.int64)
        dur = (t[:, 2] - t[:, 1]) / 1e3
        runs.append((smid, tiles, dur))
per = np.array([r[2] / r[1] for r in runs])  # us per tile, [run][cta]
print("tiles per CTA: min %d max %d" % (runs[0][1].min(), runs[0][1].max()))
print("same SM for a CTA in every run:", all(np.array_equal(runs[0][0], r[0]) for r in runs))
print("us/tile: mean %.3f  spread (max/min) %.3f" % (per.mean(), per.mean(0).max() / per.mean(0).min()))
cc = np.corrcoef(per)
print("correlation of us/tile across runs:\n", np.round(cc, 2))
order = np.argsort(per.mean(0))
print("fastest CTAs (cta, sm, us/tile):", [(int(i), int(runs[0][0][i]), round(float(per.mean(0)[i]), 3)) for i in order[:8]])
print("slowest CTAs (cta, sm, us/tile):", [(int(i), int(runs[0][0][i]), round(float(per.mean(0)[i]), 3)) for i in order[-8:]])
json.dump({"us_per_tile_mean_by_cta": per.mean(0).tolist(), "smid": runs[0][0].tolist(),
           "tiles": runs[0][1].tolist(), "corr": cc.tolist()},
          open(os.path.join(ROOT, "gpurun_out", "sm_speed.json"), "w"))
