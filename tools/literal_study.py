"""fp64 GPU vs the reference's literal fp64 path on ALL 64 BASELINE config-1 instances.

North_star's fp64 bar: recovered supports identical on >= 99 % of instances and
x_r RMSE within 1e-6 relative, against the reference's fp64 CPU path on
identical seeded inputs.  The reference path here is the oracle's LITERAL mode
(matrix-free A^T(A w), sequential, no FMA), which tests/test_ref_solver.py pins
BIT FOR BIT to the reference's own alternating_minimize compiled from
/root/reference.  Input: the fp64 GPU solve of config 1 (gpurun_out/f64_config1.npz
written by tools/r02_experiments.py / bench-side tooling); replica 0 of every
instance (the reference CLI's own stream, mix_seed(s, 1)) is re-solved here on
the host cores.
  python tools/literal_study.py gpurun_out/f64_config1.npz profiles/r02_literal_study.json
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
    src = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "gpurun_out", "f64_config1.npz")
    out_path = sys.argv[2] if len(sys.argv) > 2 else os.path.join(ROOT, "profiles",
                                                                   "r02_literal_study.json")
    d = np.load(src)
    R_gpu, S_gpu, seeds = d["R"], d["sigma"], d["seeds"]
    B = R_gpu.shape[0]
    insts = [O.gen_instance(2000, 0.5, 0.1, 0.01, 1 + b) for b in range(B)]
    sd = np.array([int(seeds[b, 0]) for b in range(B)], np.uint64)
    assert all(int(sd[b]) == O.mix_seed(1 + b, 1) for b in range(B))
    hp = O.baseline_params()
    t0 = time.perf_counter()
    _, R, S, FA = O.solve_batch(insts, sd, hp, os.cpu_count() or 1, mode=O.LITERAL)
    wall = time.perf_counter() - t0
    same = np.array([np.array_equal(S[b], S_gpu[b, 0]) for b in range(B)])
    rm_ref = np.array([O.rmse(R[b], S[b], insts[b].x_true, insts[b].xi_true) for b in range(B)])
    rm_gpu = np.array([O.rmse(R_gpu[b, 0], S_gpu[b, 0], insts[b].x_true, insts[b].xi_true)
                       for b in range(B)])
    rel = np.abs(rm_gpu - rm_ref) / rm_ref
    res = {
        "what": ("fp64 GPU solve (replica 0 of each config-1 instance) vs the oracle's LITERAL "
                 "restatement of the reference (bitwise the reference's own code, "
                 "tests/test_ref_solver.py), full schedule 20 x 1000 steps"),
        "gpu_result": os.path.basename(src), "instances": B,
        "identical_support": float(same.mean()), "identical_count": int(same.sum()),
        "rmse_rel_max": float(rel.max()), "rmse_rel_max_where_identical":
            float(rel[same].max()) if same.any() else None,
        "bar": {"identical_support_min": 0.99, "rmse_rel_max": 1e-6},
        "pass": bool(same.mean() >= 0.99 and (rel[same].max() if same.any() else 1) <= 1e-6),
        "failed": [int((FA >= 0).sum())], "cpu_wall_s": wall, "threads": os.cpu_count(),
        "differing_instances": [int(b) for b in np.nonzero(~same)[0]],
    }
    with open(out_path, "w") as f:
        json.dump(res, f, indent=1)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
