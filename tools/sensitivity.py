"""Oracle self-sensitivity: how much do fp64 supports and
RMSE depend on the G*w summation order?  Runs the same trials with the three
coupling modes (reference-literal matrix-free A^T(A w), canonical GPU order,
explicit sequential G w) and reports agreement.  CPU only (oracle)."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from oracle import oracle as O  # noqa: E402


def run(N, alpha, a, ntrial, velo, threads, out):
    insts = [O.gen_instance(N, alpha, a, 0.01, s) for s in range(1, ntrial + 1)]
    hp = O.baseline_params(velo=velo)
    seeds = np.array([O.mix_seed(i.seed, 1) for i in insts], np.uint64)
    res = {}
    for name, mode in (("literal", O.LITERAL), ("canon", O.CANON), ("explicit", O.EXPLICIT)):
        t = time.time()
        wall, R, S, FA = O.solve_batch(insts, seeds, hp, threads, mode=mode)
        res[name] = (R, S, FA)
        print(name, f"{time.time() - t:.1f}s", file=sys.stderr)
    rm = {k: [O.rmse(v[0][t], v[1][t], insts[t].x_true, insts[t].xi_true) for t in range(ntrial)]
          for k, v in res.items()}
    rep = {"N": N, "alpha": alpha, "a": a, "trials": ntrial, "velo": velo}
    for a_, b_ in (("canon", "literal"), ("explicit", "literal"), ("canon", "explicit")):
        same = int(sum(np.array_equal(res[a_][1][t], res[b_][1][t]) for t in range(ntrial)))
        rel = [abs(rm[a_][t] - rm[b_][t]) / rm[b_][t] for t in range(ntrial)]
        rep[f"{a_}_vs_{b_}"] = {"identical_supports": same, "max_rel_drmse": max(rel),
                                "mean_rel_drmse": float(np.mean(rel))}
    rep["mean_rmse_literal"] = float(np.mean(rm["literal"]))
    print(json.dumps(rep))
    with open(out, "a") as f:
        f.write(json.dumps(rep) + "\n")


if __name__ == "__main__":
    out = "profiles/sensitivity_r01.jsonl"
    run(500, 0.6, 0.2, 16, 19, 8, out)     # config 0 shape, 16 seeds
    run(2000, 0.5, 0.1, 8, 19, 8, out)     # config 1 shape, 8 instances
