"""Which fp32 quantity moves the fp64 answer?  (CPU, oracle CANON mode)

BASELINE config-1 instances (N=2000, 20 x 1000 steps, replica 0 seeds), solved
by the fp64 oracle with its precision knob (oracle.c orc_set_perturb): the local
field, the state (c, e) or the refit R rounded to fp32 at every update.  The
fraction of trajectories whose final support equals the unperturbed run says
which part of an fp32 pipeline the support-identity bar is sensitive to.
  python tools/precision_study.py [n_instances] [out.json]
"""
from __future__ import annotations

import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import oracle as O  # noqa: E402


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 16
    out_path = sys.argv[2] if len(sys.argv) > 2 else os.path.join(ROOT, "profiles",
                                                                   "r02_precision_study.json")
    insts = [O.gen_instance(2000, 0.5, 0.1, 0.01, s) for s in range(1, n + 1)]
    seeds = np.array([O.mix_seed(s, 1) for s in range(1, n + 1)], np.uint64)
    hp = O.baseline_params()
    L = O.lib()
    L.orc_set_perturb.argtypes = [O.C.c_int]
    threads = os.cpu_count() or 1
    runs = {}
    names = {0: "fp64", 1: "field_f32", 2: "state_f32", 4: "refit_R_f32", 7: "all_f32",
             8: "field_noise_2^-20", 16: "field_noise_2^-16"}
    modes = [int(m) for m in os.environ.get("MODES", "0,1,2,4,7,8,16").split(",")]
    for mode in modes:
        L.orc_set_perturb(mode)
        t0 = time.perf_counter()
        _, R, S, FA = O.solve_batch(insts, seeds, hp, threads, mode=O.CANON)
        runs[mode] = (R, S, FA)
        print(names[mode], f"{time.perf_counter() - t0:.0f}s", flush=True)
    L.orc_set_perturb(0)
    R0, S0, _ = runs[0]
    res = {"instances": n, "schedule": "config 1: 20 x 1000 steps, linear pump, Jacobi",
           "mode": "oracle CANON (fp64), replica-0 seeds", "threads": threads}
    for mode, (R, S, FA) in runs.items():
        same = np.all(S == S0, axis=1)
        rm = [O.rmse(R[k], S[k], insts[k].x_true, insts[k].xi_true) for k in range(n)]
        res[names[mode]] = {"identical_support": float(same.mean()),
                            "mean_rmse": float(np.mean(rm)), "failed": int((FA >= 0).sum())}
    with open(out_path, "w") as f:
        json.dump(res, f, indent=1)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
