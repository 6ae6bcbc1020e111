"""Quick device-timing probe of the solve on config-1 shapes (dev tool)."""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2405_00366_b200 as P  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--B", type=int, default=64)
ap.add_argument("--R", type=int, default=16)
ap.add_argument("--N", type=int, default=2000)
ap.add_argument("--alpha", type=float, default=0.5)
ap.add_argument("--a", type=float, default=0.1)
ap.add_argument("--velo", type=int, default=1)
ap.add_argument("--steps", type=int, default=1000)
ap.add_argument("--dtype", default="f32")
ap.add_argument("--graphs", type=int, default=1)
args = ap.parse_args()

t0 = time.time()
insts = P.gen_instances(args.N, [(args.alpha, args.a, 0.01, s + 1) for s in range(args.B)])
print(f"gen {time.time() - t0:.2f}s", file=sys.stderr)
hp = P.baseline_params(velo=args.velo, n_steps=args.steps)
with P.Context(0, args.dtype) as ctx:
    ctx.set_option("use_graphs", args.graphs)
    ctx.set_problems(insts)
    ctx.build_coupling()
    tg = ctx.timing()["gram_ms"]
    seeds = P.replica_seeds(insts, args.R, "mfz-bn")
    for rep in range(2):
        t1 = time.time()
        res = ctx.solve(args.R, "mfz-bn", hp, seeds)
        wall = time.time() - t1
        tm = ctx.timing()
    nalt = args.velo + 1
    step_ms = tm["cim_ms"] / (nalt * args.steps)
    es = 4 if args.dtype == "f32" else 8
    bytes_step = args.B * args.N * args.N * es
    out = dict(dtype=args.dtype, B=args.B, R=args.R, N=args.N, gram_ms=tg, wall_s=wall,
               total_ms=tm["total_ms"], cim_ms=tm["cim_ms"], refit_ms=tm["refit_ms"],
               score_ms=tm["score_ms"], step_us=step_ms * 1e3,
               step_GBps=bytes_step / (step_ms * 1e-3) / 1e9,
               spin_steps_per_s=args.B * args.R * args.N * args.steps * nalt / (tm["total_ms"] * 1e-3),
               fails=int((res["fail_alt"] >= 0).sum()),
               mean_rmse=float(np.mean(res["history"][:, :, nalt - 1]["rmse"])))
    print(json.dumps(out))
