#!/usr/bin/env python
"""Headline benchmark: MF-CIM spin-steps/s on BASELINE.json config 1.

Workload (one "step" of this script = one full pass of the hot path over the
batch): 64 seeded gen_instance(N=2000, alpha=0.5, a=0.1, nu=0.01) instances x
16 replicas, K1 gram build, 20 alternations (velo=19) x 1000 fused Euler
steps (dt 0.01, linear pump 0 -> 1.2) + damped-Jacobi refit (100 sweeps) +
scoring.  Inputs (A, y) are resident in HBM when the timed region starts;
the gram (0.57 GB of fp16 hi/lo tiles, 1.1 GB of fp64 tiles) is larger than
L2, so no flush is needed.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                  [--dtype f32|f64] [--config 0..4]

--gpus N without torchrun relaunches this script under torch.distributed.run
with N ranks (one per GPU).  Config 1 is weak-scaled (every rank solves its
own 64-instance batch, seeds offset by rank); with N > 1 a strong-scaled
sub-line splits ONE 64-instance batch across the ranks (instance shards, no
data-path collective).  Step times are the max over ranks.  ``--impl
reference`` times the reference's OWN solver (alternating_minimize compiled
from /root/reference into oracle/_ref/libref_solver.so) on the host cores, on
a bounded sample of the same workload; it never loads the CUDA library.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

CFG = dict(N=2000, alpha=0.5, a=0.1, nu=0.01, B=64, R=16, velo=19, n_steps=1000)
WORKLOADS = {
    0: "BASELINE config 0: N=500 M=300 K=100, 1 instance x 1 replica, fp64, 20 x 1000 steps",
    1: "BASELINE config 1: N=2000 M=1000 K=200 (alpha 0.5, a 0.1, nu 0.01), 64 instances x 16 "
       "replicas, 20 alternations x 1000 Euler steps, dt 0.01, linear pump 0->1.2, Jacobi refit",
    2: "BASELINE config 2: phase sweep N=2000, alpha 0.3..0.9 x a 0.05..0.3 x 32 trials = 1344 "
       "instances x 8 replicas, 20 x 1000 steps",
    3: "BASELINE config 3: MRI-shaped synthetic, N=16384 (3-level Haar of a 128x128 ellipse "
       "phantom), M=6554 random DCT rows, 1 instance x 16 replicas, 20 x 1000 steps",
    4: "BASELINE config 4 (single-GPU point of the strong-scaling run): gen_instance(N, 0.5, "
       "0.05, 0.01, 7), N=100000 M=50000 K=5000, 1 instance x 4 replicas, 10 alternations x "
       "500 steps",
}
METRIC = "MF-CIM spin-steps/s"
UNIT = "spin-steps/s"


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


READ_PEAK_PROBE_GBS = 7230.0  # profiles/r02_bulk_probe.json (chunk 65536, 148 CTAs, 128 KB in flight)


def tensor_peak_tf32():
    """Half the measured bf16 tensor rate (MEASURED_PEAKS.json), the TF32 denominator."""
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            return float(json.load(f)["bf16_tflops"]) / 2
    except Exception:
        return 2250.0 / 2  # the profiling recipe's nominal bf16 figure


def ncu_traffic(dtype="f32"):
    """Per-launch DRAM traffic of the dominant (tile) kernel from the committed ncu
    --set full captures (profiles/r02e_ncu_sym_step.json: sym_step_kernel;
    profiles/r02_ncu_sym64_step.json: sym64_step_kernel)."""
    p = os.path.join(ROOT, "profiles",
                     "r02e_ncu_sym_step.json" if dtype == "f32" else "r02_ncu_sym64_step.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return d.get("dram_bytes_per_launch")
    return None


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.samples = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(
                    ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                     "--format=csv,noheader,nounits"], capture_output=True, text=True,
                    timeout=5).stdout.strip()
                if out:
                    self.samples.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for s in self.samples for k in range(4)
                          if len(s) > 2 + k and s[2 + k].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.samples)}


def ctx_nr(R, dtype, N=2000):
    """Replica slots of a context: a power of two (>= 8 on the tensor-core path)."""
    p = 1
    while p < R:
        p *= 2
    return max(8, p) if N > 512 else p


def kernel_label(N, NR, dtype):
    """The dominant kernel of the run (runtime.cu dispatch: cluster_ok / launch_gemv)."""
    if N <= 512 and NR <= (4 if dtype != "f32" else 8):
        t = "float" if dtype == "f32" else "double"
        return (f"cluster_loop_kernel<{t},{NR},BN> (whole 1000-step CIM call per launch, G "
                "register-resident, w over DSMEM; bound by the per-step FMA chain + DSMEM "
                "round trip, so the HBM fraction is an HBM-equivalent figure)")
    if dtype == "f32":
        return (f"sym_step_kernel<{NR},BN> + sym_update_kernel<{NR},BN> (one fused "
                "Euler step: upper-triangle gram tiles as fp16 hi/lo, each read once for G w "
                "and G^T w on tcgen05; achieved counts the stored triangle bytes one step must "
                "read, dense_equivalent the dense fp32 gram share of SURVEY 8(d))")
    if N > 512:
        return (f"sym64_step_kernel<{NR},BN> + sym64_update_kernel<{NR},BN> (one fused fp64 "
                "Euler step: upper-triangle 64x64 fp64 gram tiles, each read once for G w and "
                "G^T w on the FP64 tensor cores, mma.sync m8n8k4 DMMA; bound by the DMMA pipe: "
                "achieved = 2 N^2 R flops per instance per step)")
    return f"gemv_fused_kernel<double,{NR},BN> (fused Euler step, fp64 DFMA)"


def make_instances(rank, config=1, ws=1, shard_batch=False):
    """(instances, replicas, hyper-params, default dtype) of a BASELINE config.
    Config 1 is weak-scaled (each rank its own 64 instances) unless
    shard_batch (the strong-scaled sub-line: ONE 64-instance batch split into
    contiguous blocks); config 2's fixed 1344-instance sweep is split into
    cost-balanced contiguous blocks."""
    from paper_2405_00366_b200 import workloads as W
    from paper_2405_00366_b200 import sharding
    if config == 0:
        return W.config0()
    if config == 2:
        grid = W.config2_grid()
        costs = [sharding.instance_cost(2000, int(a * 2000 + 0.5), 1000, 20)
                 for a, _, _, _ in grid]
        return W.config2(shard=sharding.instance_shard(costs, ws, rank))
    if config == 3:
        return W.config3()
    if config == 4:
        if ws > 1:
            return shared_config4(rank, ws)
        return W.config4(N=CFG.get("n4", 100_000))
    if shard_batch:
        from paper_2405_00366_b200 import cimcs
        part = sharding.instance_shard([1.0] * CFG["B"], ws, rank)
        insts = cimcs.gen_instances(2000, [(0.5, 0.1, 0.01, 1 + s) for s in part])
        return insts, CFG["R"], cimcs.baseline_params(), DEFAULT_DTYPE[1]
    insts, R, hp, _ = W.config1(rank, CFG["B"])
    return insts, R, hp, DEFAULT_DTYPE[1]


def shared_config4(rank, ws):
    """Config 4 under torchrun: the one instance (A alone is 40 GB at full size) is
    generated once, by rank 0, into /dev/shm and memory-mapped by every rank (one
    copy in the page cache instead of ws generators and ws copies); falls back to
    per-rank generation when /dev/shm cannot hold it."""
    import torch.distributed as dist
    from paper_2405_00366_b200 import workloads as W
    from paper_2405_00366_b200.cimcs import Instance
    N = CFG.get("n4", 100_000)
    d = f"/dev/shm/cimcs_c4_{N}_{os.environ.get('MASTER_PORT', '0')}"
    ok = [False]
    if rank == 0:
        insts, R, hp, dt = W.config4(N=N)
        try:
            os.makedirs(d, exist_ok=True)
            i = insts[0]
            for name, arr in (("A", i.A), ("y", i.y), ("x", i.x_true), ("xi", i.xi_true)):
                np.save(os.path.join(d, name + ".npy"), np.asfortranarray(arr))
            ok = [True]
        except OSError as e:
            print(f"config 4: /dev/shm sharing failed ({e}); ranks generate their own copy",
                  file=sys.stderr)
    dist.broadcast_object_list(ok, src=0)
    if rank == 0:
        out = insts, R, hp, dt
    elif ok[0]:
        _, R, hp, dt = W.config4(N=8)  # schedule and replica count only
        ld = lambda n: np.load(os.path.join(d, n + ".npy"), mmap_mode="r")  # noqa: E731
        inst = Instance(ld("A"), np.array(ld("y")), np.array(ld("x")), np.array(ld("xi")),
                        0.05, 0.5, 0.01, 7)
        out = [inst], R, hp, dt
    else:
        out = W.config4(N=N)
    dist.barrier()
    if rank == 0 and ok[0]:
        import shutil
        shutil.rmtree(d, ignore_errors=True)  # mapped pages stay valid until unmapped
    return out


def oracle_instances(config, n):
    """The first n instances of a BASELINE config from the ORACLE's generator
    (bit-identical to the reference's gen_instance, tests/test_pins.py): the
    reference arm never loads the product library."""
    from oracle import oracle as O
    if config == 0:
        return [O.gen_instance(500, 0.6, 0.2, 0.01, 0)], 1
    if config == 2:
        out, idx = [], 0
        for alpha in (0.3, 0.4, 0.5, 0.6, 0.7, 0.8, 0.9):
            for a in (0.05, 0.1, 0.15, 0.2, 0.25, 0.3):
                for _ in range(32):
                    if len(out) < n:
                        out.append(O.gen_instance(2000, alpha, a, 0.01, 1 + idx))
                    idx += 1
        return out, 8
    return [O.gen_instance(2000, 0.5, 0.1, 0.01, 1 + s) for s in range(n)], 16


def reference_sample(insts, nthreads, n_steps, alternations=2):
    """Bounded CPU sample on `nthreads` host threads, one trajectory per thread
    (the reference's run_jobs pool, tools/main.cpp:305-321): the reference's own
    alternating_minimize(make_problem(inst)) (orchestrator.cpp:170-235, compiled
    unmodified against the sequential Eigen shim, oracle/_ref/libref_solver.so)
    for `alternations` alternations of n_steps Euler steps + 100-sweep Jacobi
    refit + scoring.  Falls back to the oracle's LITERAL restatement (bitwise the
    same arithmetic, tests/test_ref_solver.py) when the .so is absent.
    Returns (spin-steps/s, wall_s, threads, kind)."""
    from oracle import oracle as O
    from oracle import ref_solver as RS
    use_ref = RS.available(fast=True)
    if use_ref:
        RS.use_fast(True)
    # the reference's own schedule object: its only pump is the sigmoid
    # (orchestrator.cpp:12-14); the linear ramp of the BASELINE configs is a
    # builder extension with the same per-step cost
    hp = O.HyperParams(dt=0.01, n_steps=n_steps, velo=alternations - 1)
    sel = [insts[k % len(insts)] for k in range(nthreads)]
    seeds = [O.mix_seed(i.seed, 1 + 3 * (k // len(insts))) for k, i in enumerate(sel)]
    ready = threading.Barrier(nthreads + 1)
    done = threading.Barrier(nthreads + 1)

    def one(k):
        ready.wait()
        if use_ref:
            RS.alternating_minimize(sel[k], O.MFZ_BN, hp, seeds[k])
        else:
            O.Problem(sel[k], O.LITERAL).alternating_minimize(O.MFZ_BN, hp, O.Rng(seeds[k]))
        done.wait()

    th = [threading.Thread(target=one, args=(k,)) for k in range(nthreads)]
    for t in th:
        t.start()
    ready.wait()
    t0 = time.perf_counter()
    done.wait()
    wall = time.perf_counter() - t0
    for t in th:
        t.join()
    units = sum(i.N for i in sel) * n_steps * alternations
    return units / wall, wall, nthreads, "reference" if use_ref else "port"


def cpu_sample_steps(inst, nthreads, n_steps):
    """Config 4 CPU sample: nthreads trajectories x n_steps Euler steps of run_mfz
    with the reference's matrix-free A^T(A w) (no refit: its k x k gram alone is
    O(M k^2)).  One oracle problem per thread (its LITERAL scratch is per problem,
    A is shared read-only); only the steps are timed (ctypes releases the GIL)."""
    from oracle import oracle as O
    hp = O.baseline_params(velo=1, n_steps=n_steps)
    oi = O.Instance(inst.A, inst.y, inst.x_true, inst.xi_true)
    ready = threading.Barrier(nthreads + 1)
    done = threading.Barrier(nthreads + 1)

    def one(k):
        p = O.Problem(oi, O.LITERAL)
        R = p.hz.copy()
        ready.wait()
        p.run_mfz(R, hp, 0.8, O.MFZ_BN, O.Rng(O.mix_seed(inst.seed, 1 + 3 * k)))
        done.wait()

    th = [threading.Thread(target=one, args=(k,)) for k in range(nthreads)]
    for t in th:
        t.start()
    ready.wait()
    t0 = time.perf_counter()
    done.wait()
    wall = time.perf_counter() - t0
    for t in th:
        t.join()
    return nthreads * inst.N * n_steps / wall, wall, nthreads


def ref_sample_text(n, kind, n_steps, alternations, wall, config):
    what = ("the reference's own alternating_minimize (orchestrator.cpp:170-235) compiled "
            "from /root/reference against the Eigen shim, AVX2/FMA with reassociated "
            "(vectorised) reductions as Eigen's SIMD kernels do (oracle/_ref/"
            "libref_solver_simd.so)" if kind == "reference"
            else "the oracle's LITERAL restatement of the reference (bitwise equal to it)")
    return (f"{n} trajectories (1 per host thread, distinct BASELINE config-{config} instances, "
            f"replica 0) x {alternations} alternations x {n_steps} Euler steps + 100-sweep "
            f"Jacobi refit + scoring, fp64 matrix-free A^T(A w), {what}; sigmoid pump (the "
            f"reference's only pump, same per-step cost as the linear ramp); {wall:.1f}s wall")


def run_reference(args, ws, rank):
    if rank != 0:
        return
    if args.config not in (0, 1, 2):
        print(json.dumps({"impl": "reference", "unavailable":
                          f"the reference arm covers BASELINE configs 0-2 (asked: {args.config})"}))
        return
    nthreads = os.cpu_count() or 1
    insts, _ = oracle_instances(args.config, nthreads)
    n_steps = 1000
    vals, walls, kind = [], [], "port"
    for k in range(args.warmup + args.steps):
        v, wall, n, kind = reference_sample(insts, nthreads, n_steps)
        if k >= args.warmup:
            vals.append(v)
            walls.append(wall)
    v = statistics.median(vals)
    sample = ref_sample_text(nthreads, kind, n_steps, 2, statistics.median(walls), args.config)
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": UNIT,
        "n_gpus": max(ws, args.gpus), "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * statistics.median(walls), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded gen_instance, datagen.cpp:15-55)",
        "config": {"workload": WORKLOADS[args.config], "sample": sample,
                   "same_config_note": ("bounded sample of the workload: the throughput "
                                        "metric is per spin-step, so it is comparable; the "
                                        "full config-1 job would take hours on the host")},
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": nthreads, "kind": kind,
                         "sample": sample},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# Headline dtype per config: config 1's line is the fp32 tensor-core path held
# to the declared fp32 tolerance below, with the bitwise fp64 path measured
# beside it in the same run ("f64" sub-line); config 0 is the fp64 CPU workload.
DEFAULT_DTYPE = {0: "f64", 1: "f32", 2: "f32", 3: "f32", 4: "f32"}
# fp32-mode tolerance (declared in DESIGN.md section 5 before the round-2
# measurements): against the fp64 path on the same seeded inputs.
F32_TOL = {"rmse_mean_rel": 1e-2, "hamming_mean_rel": 1e-2, "best_rmse_mean_rel": 1e-2,
           "paired_se_max": 4.0, "where_same_rmse_rel": 1e-5}


def final_metrics(res):
    B, R = res["fail_alt"].shape
    H, nh = res["history"], res["n_hist"]
    last = lambda f: np.array([[H[b, r][nh[b, r] - 1][f] if nh[b, r] else np.nan  # noqa: E731
                                for r in range(R)] for b in range(B)])
    return last("rmse"), last("hamming"), last("hamiltonian")


def parity_vs_f64(ref, res, dtype):
    """Support / quality agreement of a run with the fp64 run on the same seeds."""
    same = np.all(ref["sigma"] == res["sigma"], axis=2)
    rm0, hm0, ob0 = final_metrics(ref)
    rm1, hm1, ob1 = final_metrics(res)
    B = same.shape[0]
    b0, b1 = np.argmin(ob0, axis=1), np.argmin(ob1, axis=1)
    inst_same = np.array([np.array_equal(ref["sigma"][b, b0[b]], res["sigma"][b, b1[b]])
                          for b in range(B)])
    d = rm1 - rm0
    se = float(d.std(ddof=1) / np.sqrt(d.size)) if d.size > 1 else 0.0
    where = float(np.max(np.abs(d[same]) / rm0[same])) if same.any() else 0.0
    out = {"vs": "fp64 path, same instances and seeds", "trajectories": int(same.size),
           "traj_identical_support": float(same.mean()),
           "inst_identical_best_support": float(inst_same.mean()),
           "rmse_mean": [float(rm0.mean()), float(rm1.mean())],
           "hamming_mean": [float(hm0.mean()), float(hm1.mean())],
           "best_rmse_mean": [float(rm0[np.arange(B), b0].mean()),
                              float(rm1[np.arange(B), b1].mean())],
           "rmse_paired_diff": [float(d.mean()), se], "max_rel_rmse_where_same": where,
           "failed": [int((ref["fail_alt"] >= 0).sum()), int((res["fail_alt"] >= 0).sum())]}
    rel = lambda a: abs(a[1] - a[0]) / abs(a[0])  # noqa: E731
    out["tolerance"] = F32_TOL
    out["pass"] = bool(rel(out["rmse_mean"]) <= F32_TOL["rmse_mean_rel"]
                       and rel(out["hamming_mean"]) <= F32_TOL["hamming_mean_rel"]
                       and rel(out["best_rmse_mean"]) <= F32_TOL["best_rmse_mean_rel"]
                       and abs(d.mean()) <= F32_TOL["paired_se_max"] * max(se, 1e-300)
                       and where <= F32_TOL["where_same_rmse_rel"]
                       and out["failed"][1] <= out["failed"][0])
    return out


def gram_step_bytes(dtype, B, N):
    """Bytes one Euler step must stream: the stored gram of the path."""
    if dtype == "f32" and N > 512:
        nrb = (N + 127) // 128  # upper-triangle 128x128 tiles, fp16 hi|lo (4 B per entry)
        return B * (nrb * (nrb + 1) // 2) * 128 * 128 * 4
    if dtype == "f64" and N > 512:
        nrb = (N + 63) // 64  # upper-triangle 64x64 fp64 tiles (sym64)
        return B * (nrb * (nrb + 1) // 2) * 64 * 64 * 8
    return B * N * N * (4 if dtype == "f32" else 8)


def dmma_peak():
    """Measured FP64 tensor (DMMA) peak on this pool's B200 (tools/peaks_probe.cu)."""
    p = os.path.join(ROOT, "profiles", "r02_peaks.json")
    try:
        with open(p) as f:
            return float(json.load(f)["dmma_tflops"]), "measured (profiles/r02_peaks.json)"
    except (OSError, KeyError, ValueError):
        return 37.0, "fallback"


def measure(args, dtype, insts, R, hp, ws, rank, local, dist, tile_sharded=False,
            device_gen=None, with_e2e=True, with_dom=True):
    """One arm of the bench at one dtype: W warm-up steps, K timed steps (device
    time, max over ranks), e2e through the public API with host buffers, and
    the dominant kernel timed alone.  Returns (fields, last solve result)."""
    import paper_2405_00366_b200 as P
    import torch
    seeds = P.replica_seeds(insts, R, "mfz-bn")
    nalt = hp.velo + 1
    Bn = len(insts)
    Nn = device_gen[0] if device_gen else insts[0].N
    units = Bn * R * Nn * hp.n_steps * nalt  # spin-steps per rank per step
    if tile_sharded:
        units = units / ws

    def make_ctx():
        if not tile_sharded:
            return P.Context(local, dtype)
        nid = [P.nccl_unique_id() if rank == 0 else None]
        if dist is not None:
            dist.broadcast_object_list(nid, src=0)
        return P.Context(local, dtype, shard=(ws, rank, nid[0]))

    def load_problems(cx):
        if device_gen:
            cx.set_generated_problems(device_gen[0], device_gen[1])
        else:
            cx.set_problems(insts)

    def barrier():
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    ctx = make_ctx()
    t_gen = time.perf_counter()
    load_problems(ctx)
    torch.cuda.synchronize()
    gen_s = time.perf_counter() - t_gen

    def one_step():
        ctx.build_coupling()
        res = ctx.solve(R, "mfz-bn", hp, seeds)
        return res, ctx.timing()

    for _ in range(args.warmup):
        one_step()
    dev_ms, step_ms, launches = [], [], 0
    parts = {"gram": [], "cim": [], "refit": [], "score": []}
    barrier()
    with ClockSampler(local) as clocks:
        t0 = time.perf_counter()
        for _ in range(args.steps):
            res, tm = one_step()
            dev_ms.append(tm["gram_ms"] + tm["total_ms"])
            for k in parts:
                parts[k].append(tm[k + "_ms"])
            step_ms.append(tm["cim_ms"] / (nalt * hp.n_steps))
            launches += int(tm["step_launches"] + tm["refit_launches"] + tm["other_launches"]) + 2
        barrier()
        wall = time.perf_counter() - t0
    total_dev_ms = sum(dev_ms)
    total_units = units
    if dist is not None:
        t = torch.tensor([total_dev_ms], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_dev_ms = float(t.item())
        t = torch.tensor([float(units)], device="cuda", dtype=torch.float64)
        dist.all_reduce(t)  # config 2 / strong shards are uneven: sum what every rank did
        total_units = float(t.item())
    ms_per_step = total_dev_ms / args.steps
    value = total_units / (ms_per_step * 1e-3)

    dense_bytes = Bn * Nn * Nn * (4 if dtype == "f32" else 8)
    step_bytes = gram_step_bytes(dtype, Bn, Nn)
    if tile_sharded:
        step_bytes, dense_bytes = step_bytes / ws, dense_bytes / ws
    step_s = statistics.median(step_ms) * 1e-3
    peak, peak_kind = measured_peaks()
    achieved = step_bytes / step_s / 1e9
    # the fp64 symmetric step is bound by the FP64 tensor pipe, not HBM:
    # 2 N^2 R flops per instance per step (every replica, the whole dense G)
    f64_tensor = dtype == "f64" and Nn > 512
    step_flops = 2.0 * Bn * Nn * Nn * R

    e2e = None
    if with_e2e and not args.no_e2e:
        ctx2 = make_ctx()

        def e2e_once():
            load_problems(ctx2)
            ctx2.build_coupling()
            out = ctx2.solve(R, "mfz-bn", hp, seeds)
            torch.cuda.synchronize()
            return out

        e2e_once()  # untimed: first-use allocations and graph capture of the context
        barrier()
        times = []
        for _ in range(max(1, min(args.steps, 3))):
            t1 = time.perf_counter()
            r2 = e2e_once()
            times.append(time.perf_counter() - t1)
        ctx2.close()
        e2e_s = statistics.median(times)
        if dist is not None:
            t = torch.tensor([e2e_s], device="cuda", dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e2e_s = float(t.item())
        h2d = 0 if device_gen else sum(i.A.nbytes + i.y.nbytes + i.x_true.nbytes +
                                       i.xi_true.nbytes for i in insts)
        h2d += Bn * R * Nn * 8 * nalt  # host-drawn c0 streams
        e2e = {"value": total_units / e2e_s, "unit": UNIT, "h2d_bytes_per_step": h2d,
               "d2h_bytes_per_step": r2["R"].nbytes + r2["sigma"].nbytes +
               r2["history"].nbytes, "seconds": e2e_s}

    dom = None
    if with_dom and Nn > 512 and not tile_sharded:
        # the tile kernel alone: a short eager run with CUDA events around every
        # step-mode launch on its stream (outside the timed region)
        ctx.set_option("use_graphs", 0)
        ctx.set_option("kernel_timing", 1)
        ctx.solve(R, "mfz-bn", P.baseline_params(velo=1, n_steps=100), seeds)
        tk = ctx.timing()
        ctx.set_option("kernel_timing", 0)
        ctx.set_option("use_graphs", 1)
        if tk["tile_kernel_launches"] > 0:
            t_tile = tk["tile_kernel_ms"] / tk["tile_kernel_launches"] * 1e-3
            nr = ctx_nr(R, dtype, Nn)
            if f64_tensor:
                dp, dk = dmma_peak()
                dom = {"kernel": f"sym64_step_kernel<{nr},BN>", "bound": "tensor (FP64 DMMA)",
                       "avg_us": t_tile * 1e6, "launches": int(tk["tile_kernel_launches"]),
                       "flops_per_launch": step_flops, "achieved": step_flops / t_tile / 1e12,
                       "peak": dp, "peak_kind": dk, "unit": "TFLOP/s",
                       "frac": step_flops / t_tile / 1e12 / dp,
                       "hbm": {"bytes_per_launch": step_bytes,
                               "achieved_gbs": step_bytes / t_tile / 1e9}}
            else:
                dom = {"kernel": f"sym_step_kernel<{nr},BN>", "bound": "hbm",
                       "avg_us": t_tile * 1e6, "launches": int(tk["tile_kernel_launches"]),
                       "bytes_per_launch": step_bytes, "achieved": step_bytes / t_tile / 1e9,
                       "peak": peak, "unit": "GB/s", "frac": step_bytes / t_tile / 1e9 / peak,
                       # the driver's copy figure (read + write) understates what a pure
                       # read stream reaches: tools/bulk_probe.cu measured 7.23 TB/s for
                       # cp.async.bulk reads with 148 CTAs x 128 KB in flight
                       "read_peak_probe": {"gbs": READ_PEAK_PROBE_GBS,
                                           "frac": step_bytes / t_tile / 1e9 / READ_PEAK_PROBE_GBS,
                                           "source": "profiles/r02_bulk_probe.json"}}
            dom.update({"share_of_step": t_tile / step_s,
                        "how": ("eager run of 2 x 100 steps after the timed region, CUDA events "
                                "on the launch stream around each launch (serialised: the "
                                "kernel timed alone, burst peak)")})
    ctx.close()
    fields = {
        "value": value, "ms_per_step": ms_per_step, "steps": args.steps, "warmup": args.warmup,
        "dtype": dtype, "units_per_step": total_units,
        "instances_per_s": (Bn if tile_sharded else total_units / units * Bn) / (ms_per_step * 1e-3),
        "problem_load_s": gen_s,
        "breakdown_ms": {k: statistics.median(v) for k, v in parts.items()},
        "roofline": ({"bound": "tensor", "achieved": step_flops / step_s / 1e12,
                      "peak": dmma_peak()[0], "unit": "TFLOP/s",
                      "frac": step_flops / step_s / 1e12 / dmma_peak()[0],
                      "peak_kind_tensor": dmma_peak()[1], "hbm_achieved_gbs": achieved}
                     if f64_tensor else
                     {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                      "frac": achieved / peak}),
        "roofline_detail": {
                     "traffic": ncu_traffic(dtype) if Nn == 2000 and args.config == 1 else None,
                     "kernel": kernel_label(Nn, ctx_nr(R, dtype, Nn), dtype),
                     "bytes_per_launch": step_bytes, "peak_kind": peak_kind,
                     "step_us": step_s * 1e6, "dominant_kernel": dom,
                     "dense_equivalent": {"bytes_per_launch": dense_bytes,
                                          "achieved": dense_bytes / step_s / 1e9}},
        "e2e": e2e, "gpu_launches": launches, "clocks": clocks.summary(), "wall_s": wall,
        "l2": ("inputs larger than L2 (gram %.2f GB per step)" % (step_bytes / 1e9)
               if step_bytes > 126e6 else "gram fits in L2 (no flush)"),
    }
    fields["roofline"].update(fields.pop("roofline_detail"))
    return fields, res


def run_ours(args, ws, rank, local):
    import paper_2405_00366_b200 as P
    from paper_2405_00366_b200 import _lib
    _lib.load()  # before torch (the product library binds torch's NCCL)
    import torch

    torch.cuda.set_device(local)
    dist = None
    if ws > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl")
    device_gen = None
    if args.device_gen and args.config == 4:  # counter-based, a deviation
        from paper_2405_00366_b200.workloads import config4 as _c4
        _, R, hp, wdtype = _c4(N=8)
        Nd = CFG.get("n4", 100_000)
        device_gen = (Nd, [(0.5, 0.05, 0.01, 7)])
        Md, _ = P.gen_dims(Nd, 0.5, 0.05)
        insts = [P.Instance(np.zeros((Md, 0)), np.zeros(0), seed=7)]  # shape/seed stand-in
    else:
        insts, R, hp, wdtype = make_instances(rank, args.config, ws)
    dtype = args.dtype or (DEFAULT_DTYPE[args.config] if args.config == 1 else wdtype)
    # config 4 on several GPUs (or --shard): ONE instance split by gram tiles
    # across the ranks (tile-sharded contexts: replicated state, one NCCL
    # all-reduce per step) -- strong scaling
    tile_sharded = args.config == 4 and (ws > 1 or args.shard)
    main, res = measure(args, dtype, insts, R, hp, ws, rank, local, dist, tile_sharded,
                        device_gen)
    Nn = device_gen[0] if device_gen else insts[0].N

    extra, results = {}, {dtype: res}
    if args.config == 1 and not args.no_extra:
        # the other precisions of config 1 on the same instances and seeds, each a
        # full measurement; parity of every non-fp64 run against the fp64 run
        for dt in ("f64", "f32"):
            if dt == dtype:
                continue
            f, r = measure(args, dt, insts, R, hp, ws, rank, local, dist, with_dom=True)
            extra[dt] = f
            results[dt] = r
        par = {dt: parity_vs_f64(results["f64"], results[dt], dt)
               for dt in results if dt != "f64"}
        if dist is not None:  # every rank checked its own batch: report rank 0's, AND the passes
            ok = torch.tensor([min(int(p["pass"]) for p in par.values())], device="cuda")
            dist.all_reduce(ok, op=dist.ReduceOp.MIN)
            for p in par.values():
                p["pass_all_ranks"] = bool(ok.item())
        main["parity"] = par
        if ws > 1:  # strong scaling: ONE 64-instance batch split across the ranks
            si, sR, shp, _ = make_instances(rank, 1, ws, shard_batch=True)
            f, _ = measure(args, dtype, si, sR, shp, ws, rank, local, dist, with_e2e=False,
                           with_dom=False)
            extra["strong_scaled_batch"] = {
                "workload": "ONE config-1 batch of 64 instances split into contiguous "
                            f"instance shards over {ws} ranks (no data-path collective)",
                "scaling": "strong", "value": f["value"], "ms_per_step": f["ms_per_step"],
                "per_rank_instances": len(si)}

    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu and not device_gen:
        nthreads = os.cpu_count() or 1
        if args.config == 4:
            cs = 2
            v, wall_c, n = cpu_sample_steps(insts[0], min(nthreads, 8), cs)
            cpu = {"value": v, "unit": UNIT, "cores": n, "kind": "port",
                   "sample": (f"{n} trajectories (1/host thread) x {cs} Euler steps of run_mfz, "
                              f"fp64 A^T(A w) restatement, no refit, {wall_c:.1f}s wall")}
        elif args.config in (0, 1, 2):
            oi, _ = oracle_instances(args.config, nthreads)
            v, wall_c, n, kind = reference_sample(oi, nthreads, 1000, 2)
            cpu = {"value": v, "unit": UNIT, "cores": n, "kind": kind,
                   "sample": ref_sample_text(n, kind, 1000, 2, wall_c, args.config)}
        else:  # config 3: Euler steps of the oracle port on the MRI-shaped instance
            cs = 5
            v, wall_c, n = cpu_sample_steps(insts[0], min(nthreads, 8), cs)
            cpu = {"value": v, "unit": UNIT, "cores": n, "kind": "port",
                   "sample": (f"{n} trajectories (1/host thread) x {cs} Euler steps of run_mfz, "
                              f"fp64 A^T(A w) restatement, no refit, {wall_c:.1f}s wall")}
    if rank == 0:
        wl = WORKLOADS[args.config]
        if args.config == 4 and args.n4 != 100_000:
            wl = wl.replace("N=100000 M=50000 K=5000", f"N={Nn} (reduced)")
        line = {
            "metric": METRIC, "value": main["value"], "unit": UNIT, "n_gpus": ws,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": main["ms_per_step"],
            "higher_is_better": True,
            "scaling": "strong" if args.config == 2 or tile_sharded else "weak",
            "vs_baseline": None, "dtype": dtype,
            "data": ("synthetic, generated on the GPU from counter-based Philox streams "
                     "(documented deviation: not the reference's mt19937_64 instance)"
                     if device_gen else "synthetic (seeded gen_instance, datagen.cpp:15-55)"),
            "config": {"workload": wl, "per_rank_instances": len(insts), "replicas": R,
                       "parallelism": (f"tile-sharded gram x{ws} (replicated state, one NCCL "
                                       "all-reduce per step)" if tile_sharded else
                                       f"instance shards x{ws}"),
                       "step": "gram build + full alternating solve", "l2": main["l2"]},
        }
        for k in ("instances_per_s", "problem_load_s", "breakdown_ms", "roofline", "e2e",
                  "gpu_launches", "clocks", "wall_s", "parity"):
            if k in main:
                line[k] = main[k]
        if cpu is not None:
            line["cpu_baseline"] = cpu
        for k, f in extra.items():
            line[k] = f
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()


def run_chain3(args, ws, rank, local):
    """Config 3 through the matrix-free DCT o Haar^-1 chain (csrc/dct_kernels.cuh):
    the same instance as the dense config-3 path (same phantom, frequencies,
    observations), G never stored.  A step is hz/diag build + the full
    alternating solve (20 x 1000 steps, damped Jacobi refits on the chain).
    Replicas-only under torchrun (each rank its own seed)."""
    import torch
    import paper_2405_00366_b200 as P
    from paper_2405_00366_b200 import _lib, workloads
    _lib.load()

    torch.cuda.set_device(local)
    dist = None
    if ws > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl")
    n, L, freqs, y, w = workloads.config3_chain(seed=3 + rank)
    R, hp = 16, P.baseline_params()
    N, nalt = n * n, hp.velo + 1
    units = R * N * hp.n_steps * nalt
    seeds = np.array([[P.mix_seed(3 + rank, 1 + 3 * r) for r in range(R)]], np.uint64)

    def barrier():
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    ctx = P.Context(local, "f32")
    ctx.set_dct_problem(n, L, freqs, y, w)

    def one_step():
        ctx.build_coupling()
        return ctx.solve(R, "mfz-bn", hp, seeds), ctx.timing()

    for _ in range(args.warmup):
        one_step()
    dev_ms, step_us, launches = [], [], 0
    parts = {"gram": [], "cim": [], "refit": [], "score": []}
    barrier()
    with ClockSampler(local) as clocks:
        for _ in range(args.steps):
            res, tm = one_step()
            dev_ms.append(tm["gram_ms"] + tm["total_ms"])
            for k in parts:
                parts[k].append(tm[k + "_ms"])
            step_us.append(1e3 * tm["cim_ms"] / (nalt * hp.n_steps))
            launches += int(tm["step_launches"] + tm["refit_launches"] + tm["other_launches"]) + 2
        barrier()
    total = sum(dev_ms)
    if dist is not None:
        t = torch.tensor([total], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total = float(t.item())
    ms = total / args.steps
    value = units * ws / (ms * 1e-3)
    # the chain kernel alone (eager, CUDA events around each step launch)
    ctx.set_option("use_graphs", 0)
    ctx.set_option("kernel_timing", 1)
    ctx.solve(R, "mfz-bn", P.baseline_params(velo=1, n_steps=100), seeds)
    tk = ctx.timing()
    ctx.set_option("kernel_timing", 0)
    ctx.set_option("use_graphs", 1)
    ctx.close()
    e2e = None
    if not args.no_e2e:
        def e2e_once():
            with P.Context(local, "f32") as c2:
                c2.set_dct_problem(n, L, freqs, y, w)
                c2.build_coupling()
                out = c2.solve(R, "mfz-bn", hp, seeds)
            torch.cuda.synchronize()
            return out
        e2e_once()
        barrier()
        times = []
        for _ in range(max(1, min(args.steps, 3))):
            t1 = time.perf_counter()
            r2 = e2e_once()
            times.append(time.perf_counter() - t1)
        e2e_s = statistics.median(times)
        if dist is not None:
            t = torch.tensor([e2e_s], device="cuda", dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e2e_s = float(t.item())
        h2d = freqs.nbytes + y.nbytes + w.nbytes + 2 * N * 4 + N + R * N * 8 * nalt
        e2e = {"value": units * ws / e2e_s, "unit": UNIT, "h2d_bytes_per_step": h2d,
               "d2h_bytes_per_step": r2["R"].nbytes + r2["sigma"].nbytes + r2["history"].nbytes,
               "seconds": e2e_s}
    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu:
        insts, _, _, _ = workloads.config3()  # the dense instance the reference would run
        nthreads = os.cpu_count() or 1
        cs = 5
        v, wall_c, k = cpu_sample_steps(insts[0], min(nthreads, 8), cs)
        cpu = {"value": v, "unit": UNIT, "cores": k, "kind": "port",
               "sample": (f"{k} trajectories (1/host thread) x {cs} Euler steps of run_mfz on "
                          f"the dense config-3 instance, fp64 A^T(A w) restatement, no refit, "
                          f"{wall_c:.1f}s wall")}
    if rank == 0:
        st = statistics.median(step_us)
        t_k = tk["tile_kernel_ms"] / max(1, tk["tile_kernel_launches"]) * 1e-3
        fl = 4 * 2.0 * n ** 3 * 3 * R  # 4 slab products x 3 TF32 passes per vector
        rm = [res["history"][0, r][res["n_hist"][0, r] - 1]["rmse"] for r in range(R)]
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (workloads.config3_chain: the config-3 phantom, frequencies, noise)",
            "config": {"workload": WORKLOADS[3] + " -- matrix-free DCT o Haar^-1 chain, G never "
                                   "stored",
                       "step": "hz/diag build + full alternating solve (20 x 1000, Jacobi refit)",
                       "l2": "no gram: DCT matrix + 16 images, L2/SMEM resident (no flush)"},
            "breakdown_ms": {k: statistics.median(v) for k, v in parts.items()},
            "roofline": {"bound": "tensor",
                         # 3xTF32 flops of the four slab products vs HALF the measured bf16
                         # tensor rate (TF32 = half the bf16 rate; no TF32 figure is measured
                         # on this pool): a small fraction -- the step is latency-bound
                         "achieved": fl / (st * 1e-6) / 1e12, "unit": "TFLOP/s",
                         "peak": tensor_peak_tf32(), "frac": fl / (st * 1e-6) / 1e12 / tensor_peak_tf32(),
                         "traffic": None, "latency_bound": True,
                         "note": ("one 8-CTA cluster per replica: 4 slab products 16x128x128 on "
                                  "mma.sync TF32 (3xTF32), 2 DSMEM all-gathers, Haar in the slab;"
                                  " no HBM stream"),
                         "step_us": st, "chain_kernel_us": t_k * 1e6,
                         "chain_tflops": fl / t_k / 1e12 if t_k > 0 else None,
                         "kernel": "dct_cluster_kernel + sym_update_kernel<16,BN>",
                         "dense_path_step_us": 120.0},
            "e2e": e2e, "final_rmse_median": float(np.median(rm)),
            "gpu_launches": launches, "clocks": clocks.summary(),
        }
        if cpu is not None:
            line["cpu_baseline"] = cpu
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()


def run_mri(args, ws, rank, local):
    """--mri: the reference's own transform-chain MRI problem (mri.cpp, cmd_mri
    tools/main.cpp:506-560) at config-3 size, matrix-free on the GPU
    (csrc/mri_kernels.cuh): 128x128 phantom sparsified to 10 % of its Haar
    coefficients, 40 % random k-space samples, gamma 1e-4, 16 replicas, 20 x
    1000 Euler steps with the BASELINE pump, CG refits.  A step is the whole
    solve; replicas-only under torchrun (each rank its own mask seed)."""
    import torch
    import paper_2405_00366_b200 as P
    from paper_2405_00366_b200 import mri as PM

    torch.cuda.set_device(local)
    dist = None
    if ws > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl")
    size, R = 128, 16
    img, coeffs, mask = PM.problem(size, 0.1, 0.4, 1 + rank)
    hp = P.baseline_params()
    nalt = hp.velo + 1
    N = size * size
    units = R * N * hp.n_steps * nalt
    seeds = np.array([[P.mix_seed(1 + rank, 1 + 3 * r) for r in range(R)]], np.uint64)
    ctx = P.Context(local, "f32")

    def one_step():
        ctx.set_mri_problem(img, mask, 1e-4, coeffs)
        ctx.build_coupling()
        t0 = time.perf_counter()
        x0, _, _ = ctx.mri_lasso(3e-4)  # cmd_mri's warm start lasso_init (main.cpp:532)
        tl = time.perf_counter() - t0
        r0 = np.broadcast_to(x0, (1, R, N)).copy()
        res = ctx.solve(R, "mfz-bn", hp, seeds, R_init=r0)
        tm = ctx.timing()
        tm["lasso_ms"] = 1e3 * tl
        return res, tm

    for _ in range(args.warmup):
        one_step()

    def barrier():
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    dev_ms, step_us, launches = [], [], 0
    barrier()
    with ClockSampler(local) as clocks:
        for _ in range(args.steps):
            res, tm = one_step()
            dev_ms.append(tm["gram_ms"] + tm["lasso_ms"] + tm["total_ms"])
            step_us.append(1e3 * tm["cim_ms"] / (nalt * hp.n_steps))
            launches += int(tm["step_launches"] + tm["refit_launches"] + tm["other_launches"]) + 2
        barrier()
    total = sum(dev_ms)
    if dist is not None:
        t = torch.tensor([total], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total = float(t.item())
    ms = total / args.steps
    value = units * ws / (ms * 1e-3)
    ok = int((res["fail_alt"][0] < 0).sum())
    rm = [res["history"][0, r][res["n_hist"][0, r] - 1]["rmse"] for r in range(R)]
    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu:
        from oracle import mri as OM
        t0 = OM.MriTransform(img, mask, 1e-4)
        w = np.random.default_rng(0).normal(size=N)
        k, t1 = 0, time.perf_counter()
        while time.perf_counter() - t1 < 10.0:
            t0.apply_full(w)
            k += 1
        wall = time.perf_counter() - t1
        cpu = {"value": N * k / wall, "unit": UNIT, "cores": 1, "kind": "port",
               "sample": (f"{k} fp64 apply_full calls of the numpy restatement of mri.cpp "
                          f"(the per-step coupling; numpy FFT), {wall:.1f}s wall, one trajectory")}
    ctx.close()
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (the reference's phantom_image, sparsify_wavelet, make_mask)",
            "config": {"workload": ("config-3 size, the reference's own matrix-free MRI chain: "
                                    "128x128 phantom, 10 % Haar coefficients, 40 % k-space, "
                                    "gamma 1e-4, 1 x 16 replicas, LASSO warm start (lambda 3e-4), "
                                    "20 x 1000 steps, CG refit"),
                       "step": "hz/diag build + LASSO warm start (host-timed) + full alternating solve",
                       "l2": "operator applied from shared memory (no gram)"},
            "roofline": {"bound": "hbm",
                         # the step only moves the state: R, c, e read, c, e, w written and w
                         # read back (7 x N x R replicas x 4 B); the FFT chain runs from shared
                         # memory and registers -- a small fraction: the step is latency-bound
                         "achieved": 7 * N * R * 4 / (statistics.median(step_us) * 1e-6) / 1e9,
                         "unit": "GB/s", "peak": measured_peaks()[0],
                         "frac": 7 * N * R * 4 / (statistics.median(step_us) * 1e-6) / 1e9 / measured_peaks()[0],
                         "traffic": None, "latency_bound": True,
                         "note": "per-step latency of one 8-CTA cluster per replica (FFT lines "
                                 "in warp registers, row/column slabs exchanged over DSMEM, "
                                 "Haar level 1 distributed); no HBM stream",
                         "step_us": statistics.median(step_us),
                         "kernel": "mri_cluster_kernel + sym_update_kernel<16,BN>"},
            "replicas_ok": ok, "final_rmse_median": float(np.median(rm)),
            "gpu_launches": launches, "clocks": clocks.summary(),
        }
        if cpu is not None:
            line["cpu_baseline"] = cpu
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()


def relaunch(args):
    """--gpus N outside torchrun: run this script under torch.distributed.run with
    N ranks on this node (rendezvous on 127.0.0.1); rank 0 prints the line."""
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1",
           f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=None,
                    help="timed steps (default 3; 40 for the 36 ms config-0 job so the clock "
                         "sampler sees the run)")
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--dtype", default=None, choices=["f32", "f64"],
                    help="default: the config's (f32 for 1-4, f64 for 0)")
    ap.add_argument("--config", type=int, default=1, choices=[0, 1, 2, 3, 4])
    ap.add_argument("--n4", type=int, default=100_000, help="config 4 size (N)")
    ap.add_argument("--dense", action="store_true",
                    help="config 3: the dense gram path instead of the matrix-free chain")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-extra", action="store_true",
                    help="config 1: skip the other-precision lines and their parity check")
    ap.add_argument("--device-gen", action="store_true",
                    help="config 4: generate the instance on the GPU (counter-based deviation)")
    ap.add_argument("--shard", action="store_true",
                    help="config 4: use the tile-sharded context even on one GPU")
    ap.add_argument("--mri", action="store_true",
                    help="the reference's matrix-free MRI chain at config-3 size (run_mri)")
    args = ap.parse_args()
    if args.steps is None:
        args.steps = 40 if (args.config == 0 and not args.mri and args.impl == "ours") else 3
    CFG["n4"] = args.n4
    ws, rank, local = dist_env()
    if args.impl == "ours" and args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(relaunch(args))
    if args.impl == "ours" and ws != args.gpus and "WORLD_SIZE" in os.environ and rank == 0:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={ws}; measuring {ws} ranks",
              file=sys.stderr)
    if args.mri and args.impl == "ours":
        run_mri(args, ws, rank, local)
    elif args.config == 3 and args.impl == "ours" and not args.dense:
        run_chain3(args, ws, rank, local)
    elif args.impl == "reference":
        run_reference(args, ws, rank)
    else:
        run_ours(args, ws, rank, local)


if __name__ == "__main__":
    main()
