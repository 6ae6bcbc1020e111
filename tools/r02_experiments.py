"""Round-2 GPU experiments (run on the B200 box; outputs under gpurun_out/):

1. sensitivity: BASELINE config 1 (64 x 16, N=2000, 20 x 1000) solved in fp64
   twice -- with the reference's R_init = hz, and with R_init rounded to fp32
   (a perturbation at fp32 rounding level of the initial state only) -- and in
   fp32.  Reports support identity and quality metrics of each against the
   unperturbed fp64 run, and saves the fp64 replica-0 answers for the
   LITERAL-oracle study (tools/literal_study.py).
2. l2groups: fp32 config-1 instances solved in groups of g instances per
   context (gram tiles copied with evict_first / evict_last), per-step time.
"""
from __future__ import annotations

import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2405_00366_b200 as P  # noqa: E402
from paper_2405_00366_b200 import workloads as W  # noqa: E402

OUT = os.path.join(ROOT, "gpurun_out")
os.makedirs(OUT, exist_ok=True)


def final(res):
    B, R = res["fail_alt"].shape
    rm = np.array([[res["history"][b, r][res["n_hist"][b, r] - 1]["rmse"] for r in range(R)]
                   for b in range(B)])
    hm = np.array([[res["history"][b, r][res["n_hist"][b, r] - 1]["hamming"] for r in range(R)]
                   for b in range(B)])
    ob = np.array([[res["history"][b, r][res["n_hist"][b, r] - 1]["hamiltonian"]
                    for r in range(R)] for b in range(B)])
    return rm, hm, ob


def compare(ref, res):
    same = np.all(ref["sigma"] == res["sigma"], axis=2)
    rm0, hm0, ob0 = final(ref)
    rm1, hm1, ob1 = final(res)
    best0 = np.argmin(ob0, axis=1)
    best1 = np.argmin(ob1, axis=1)
    B = same.shape[0]
    inst_same = np.array([np.array_equal(ref["sigma"][b, best0[b]], res["sigma"][b, best1[b]])
                          for b in range(B)])
    d = rm1 - rm0
    return {
        "traj_identical_support": float(same.mean()),
        "inst_identical_best_support": float(inst_same.mean()),
        "rmse_mean": [float(rm0.mean()), float(rm1.mean())],
        "rmse_paired_diff_mean": float(d.mean()),
        "rmse_paired_diff_se": float(d.std(ddof=1) / np.sqrt(d.size)),
        "hamming_mean": [float(hm0.mean()), float(hm1.mean())],
        "best_rmse_mean": [float(rm0[np.arange(B), best0].mean()),
                           float(rm1[np.arange(B), best1].mean())],
        "max_rel_rmse_where_same": float(np.max(np.abs(d[same]) / rm0[same])) if same.any() else None,
        "failed": [int((ref["fail_alt"] >= 0).sum()), int((res["fail_alt"] >= 0).sum())],
    }


def sensitivity():
    insts, R, hp, _ = W.config1(0, 64)
    seeds = P.replica_seeds(insts, R, "mfz-bn")
    out = {}
    with P.Context(0, "f64") as ctx:
        ctx.set_problems(insts)
        ctx.build_coupling()
        t0 = time.perf_counter()
        ref = ctx.solve(R, "mfz-bn", hp, seeds)
        out["f64_s"] = time.perf_counter() - t0
        hz = np.stack([ctx.get_coupling(b, gram=False)[1] for b in range(len(insts))])
        r0 = np.broadcast_to(hz.astype(np.float32).astype(np.float64)[:, None, :],
                             (len(insts), R, insts[0].N)).copy()
        pert = ctx.solve(R, "mfz-bn", hp, seeds, R_init=r0)
    out["f64_rinit_f32"] = compare(ref, pert)
    with P.Context(0, "f32") as ctx:
        ctx.set_problems(insts)
        ctx.build_coupling()
        t0 = time.perf_counter()
        r32 = ctx.solve(R, "mfz-bn", hp, seeds)
        out["f32_s"] = time.perf_counter() - t0
    out["f32"] = compare(ref, r32)
    with P.Context(0, "f32") as ctx:
        ctx.set_option("tensor_cores", 0)
        ctx.set_problems(insts)
        ctx.build_coupling()
        rcc = ctx.solve(R, "mfz-bn", hp, seeds)
    out["f32_cudacore"] = compare(ref, rcc)
    np.savez_compressed(os.path.join(OUT, "f64_config1.npz"), R=ref["R"], sigma=ref["sigma"],
                        history=ref["history"], n_hist=ref["n_hist"], fail_alt=ref["fail_alt"],
                        seeds=seeds)
    with open(os.path.join(OUT, "sensitivity_r02.json"), "w") as f:
        json.dump(out, f, indent=1)
    print(json.dumps(out, indent=1))


def mixed():
    """F32X (tensor-core fp32 coupling, fp64 state) vs the fp64 path at config 1."""
    insts, R, hp, _ = W.config1(0, 64)
    seeds = P.replica_seeds(insts, R, "mfz-bn")
    out = {}
    with P.Context(0, "f64") as ctx:
        ctx.set_problems(insts)
        ctx.build_coupling()
        ref = ctx.solve(R, "mfz-bn", hp, seeds)
        out["f64_ms"] = ctx.timing()
    for dt in ("f32x", "f32"):
        with P.Context(0, dt) as ctx:
            ctx.set_problems(insts)
            ctx.build_coupling()
            ctx.solve(R, "mfz-bn", hp, seeds)
            res = ctx.solve(R, "mfz-bn", hp, seeds)
            out[dt + "_timing"] = ctx.timing()
        out[dt] = compare(ref, res)
    with open(os.path.join(OUT, "mixed_r02.json"), "w") as f:
        json.dump(out, f, indent=1)
    print(json.dumps(out, indent=1))


def f64perf():
    """fp64 config 1: DMMA symmetric path vs the CUDA-core grid kernel (sym64=0)."""
    insts, R, hp, _ = W.config1(0, 64)
    seeds = P.replica_seeds(insts, R, "mfz-bn")
    out = {}
    res = {}
    for s64 in (1, 0):
        with P.Context(0, "f64") as ctx:
            ctx.set_option("sym64", s64)
            ctx.set_problems(insts)
            ctx.build_coupling()
            ctx.solve(R, "mfz-bn", hp, seeds)
            res[s64] = ctx.solve(R, "mfz-bn", hp, seeds)
            t = ctx.timing()
            out[f"sym64={s64}"] = {k: t[k] for k in ("total_ms", "gram_ms", "cim_ms", "refit_ms")}
            out[f"sym64={s64}"]["us_per_step"] = t["cim_ms"] / 20000 * 1e3
            if s64:
                ctx.set_option("use_graphs", 0)
                ctx.set_option("kernel_timing", 1)
                ctx.solve(R, "mfz-bn", P.baseline_params(velo=1, n_steps=100), seeds)
                tk = ctx.timing()
                out["sym64_tile_kernel_us"] = tk["tile_kernel_ms"] / tk["tile_kernel_launches"] * 1e3
    out["vs_cudacore"] = compare(res[0], res[1])
    with open(os.path.join(OUT, "f64perf_r02.json"), "w") as f:
        json.dump(out, f, indent=1)
    print(json.dumps(out, indent=1))


def sym64warps():
    """DMMA tile kernel with 8 vs 16 DMMA warps: per-step time, bitwise-equal results."""
    insts, R, hp, _ = W.config1(0, 64)
    hp = P.baseline_params(velo=3, n_steps=1000)
    seeds = P.replica_seeds(insts, R, "mfz-bn")
    out, res = {}, {}
    for nw in (8, 16):
        with P.Context(0, "f64") as ctx:
            ctx.set_option("sym64_warps", nw)
            ctx.set_problems(insts)
            ctx.build_coupling()
            ctx.solve(R, "mfz-bn", hp, seeds)
            res[nw] = ctx.solve(R, "mfz-bn", hp, seeds)
            t = ctx.timing()
            out[nw] = {"us_per_step": t["cim_ms"] / 4000 * 1e3, "refit_ms": t["refit_ms"]}
            ctx.set_option("use_graphs", 0)
            ctx.set_option("kernel_timing", 1)
            ctx.solve(R, "mfz-bn", P.baseline_params(velo=1, n_steps=100), seeds)
            tk = ctx.timing()
            out[nw]["tile_us"] = tk["tile_kernel_ms"] / tk["tile_kernel_launches"] * 1e3
    out["bitwise_equal"] = bool(np.array_equal(res[8]["R"], res[16]["R"]) and
                                np.array_equal(res[8]["sigma"], res[16]["sigma"]))
    print(json.dumps(out, indent=1))


def refitcmp():
    """fp32 config 1: full vs compacted Jacobi refit -- time and parity vs fp64."""
    import bench
    insts, R, hp, _ = W.config1(0, 64)
    seeds = P.replica_seeds(insts, R, "mfz-bn")
    out = {}
    with P.Context(0, "f64") as ctx:
        ctx.set_problems(insts)
        ctx.build_coupling()
        ref = ctx.solve(R, "mfz-bn", hp, seeds)
    for cmp in (0, 1):
        with P.Context(0, "f32") as ctx:
            ctx.set_option("refit_compact", cmp)
            ctx.set_problems(insts)
            ctx.build_coupling()
            ctx.solve(R, "mfz-bn", hp, seeds)
            res = ctx.solve(R, "mfz-bn", hp, seeds)
            t = ctx.timing()
        par = bench.parity_vs_f64(ref, res, "f32")
        out[cmp] = {k: t[k] for k in ("total_ms", "cim_ms", "refit_ms", "score_ms")}
        out[cmp].update({k: par[k] for k in ("traj_identical_support", "rmse_mean", "hamming_mean",
                                             "rmse_paired_diff", "max_rel_rmse_where_same",
                                             "pass")})
    print(json.dumps(out, indent=1))


def l2groups():
    insts, R, hp, _ = W.config1(0, 64)
    hp1 = P.baseline_params(velo=1, n_steps=500)  # 2 x 500 steps
    seeds = P.replica_seeds(insts, R, "mfz-bn")
    rows = []
    for g in (64, 16, 8, 4):
        for keep in (0, 1):
            cim = 0.0
            for k in range(0, 64, g):
                with P.Context(0, "f32") as ctx:
                    ctx.set_problems(insts[k:k + g])
                    ctx.build_coupling()
                    ctx.set_option("gram_l2", keep)
                    ctx.solve(R, "mfz-bn", hp1, seeds[k:k + g])
                    ctx.solve(R, "mfz-bn", hp1, seeds[k:k + g])
                    cim += ctx.timing()["cim_ms"]
            rows.append({"group": g, "evict_last": keep, "us_per_step_all64": cim / 1000 * 1e3})
            print(rows[-1], flush=True)
    with open(os.path.join(OUT, "l2groups_r02.json"), "w") as f:
        json.dump(rows, f, indent=1)


def l2subset():
    """A fixed L2-resident SUBSET of the gram: the first `keep` tiles of every
    instance's triangle copied with evict_last, the rest evict_first."""
    insts, R, hp, _ = W.config1(0, 64)
    hp1 = P.baseline_params(velo=1, n_steps=500)
    seeds = P.replica_seeds(insts, R, "mfz-bn")
    rows = []
    with P.Context(0, "f32") as ctx:
        ctx.set_problems(insts)
        ctx.build_coupling()
        for keep in (0, 4, 8, 12, 16, 24, 32, 0):
            ctx.set_option("gram_l2", keep)
            ctx.solve(R, "mfz-bn", hp1, seeds)
            ts = []
            for _ in range(2):
                ctx.solve(R, "mfz-bn", hp1, seeds)
                ts.append(ctx.timing()["cim_ms"] / 1000 * 1e3)
            rows.append({"keep_tiles_per_instance": keep, "kept_MB": keep * 64 * 65536 / 1e6,
                         "us_per_step": min(ts)})
            print(rows[-1], flush=True)
    with open(os.path.join(OUT, "l2subset_r02.json"), "w") as f:
        json.dump(rows, f, indent=1)


if __name__ == "__main__":
    which = sys.argv[1:] or ["sensitivity", "l2groups"]
    for w in which:
        globals()[w]()
