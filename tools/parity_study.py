"""Parity at full BASELINE config-1 scale (64 instances x 16 replicas, N = 2000,
20 x 1000 steps): the fp32 tensor-core solve against the fp64 solve.  The fp64
GPU path is bitwise equal to the oracle's canonical-order restatement (tests/
test_gpu_parity.py, test_golden.py), so this measures fp32-vs-oracle agreement
on all 1024 trajectories, which the oracle itself could not afford on a CPU.
Prints one JSON line (profiles/r01e_parity_config1.json)."""
import json
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2405_00366_b200 as P
from paper_2405_00366_b200 import workloads as W

variant = sys.argv[1] if len(sys.argv) > 1 else "sym"  # sym | cudacore
cfg = int(sys.argv[2]) if len(sys.argv) > 2 else 1     # BASELINE config 1 or 2
insts, R, hp, _ = W.config1() if cfg == 1 else W.config2()
seeds = P.replica_seeds(insts, R, "mfz-bn")
out = {}
for dt in ("f64", "f32"):
    with P.Context(0, dt) as ctx:
        if dt == "f32" and variant == "cudacore":
            ctx.set_option("tensor_cores", 0)
        ctx.set_problems(insts)
        ctx.build_coupling()
        out[dt] = ctx.solve(R, "mfz-bn", hp, seeds)
a, b = out["f64"], out["f32"]
B = len(insts)
same = (a["sigma"] == b["sigma"]).all(axis=2)           # [B, R]
fail = (a["fail_alt"] >= 0) | (b["fail_alt"] >= 0)
last = lambda r, bb, q: r["history"][bb, q][r["n_hist"][bb, q] - 1]["rmse"]  # noqa: E731
rel = np.array([[abs(last(b, bb, q) - last(a, bb, q)) / max(last(a, bb, q), 1e-300)
                 for q in range(R)] for bb in range(B)])
# per-instance answer: the replica with the minimum final objective
def best(r):
    h = np.array([[r["history"][bb, q][r["n_hist"][bb, q] - 1]["hamiltonian"] for q in range(R)]
                  for bb in range(B)])
    return h.argmin(axis=1)
ba, bb_ = best(a), best(b)
inst_same = np.array([np.array_equal(a["sigma"][k, ba[k]], b["sigma"][k, bb_[k]]) for k in range(B)])
def quality(r):
    rm = np.array([[last(r, bb, q) for q in range(R)] for bb in range(B)])
    ham = np.array([[r["history"][bb, q][r["n_hist"][bb, q] - 1]["hamming"] for q in range(R)]
                    for bb in range(B)])
    return {"rmse_mean": float(rm.mean()), "rmse_median": float(np.median(rm)),
            "exact_support_fraction": float((ham == 0).mean()),
            "hamming_mean": float(ham.mean())}
line = {"workload": (f"BASELINE config {cfg} ({B} x {R}, N=2000, 20 x 1000 steps)"), "fp32_variant": variant,
        "quality_vs_truth": {"f64": quality(a), "f32": quality(b)},
        "trajectories": int(B * R), "failed": int(fail.sum()),
        "support_identical_trajectories": float(same.mean()),
        "support_identical_instances_best_replica": float(inst_same.mean()),
        "rmse_rel_diff_median": float(np.median(rel)), "rmse_rel_diff_mean": float(rel.mean()),
        "rmse_rel_diff_max": float(rel.max()),
        "rmse_rel_diff_identical_support_max": float(rel[same].max()) if same.any() else None}
print(json.dumps(line))
