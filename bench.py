#!/usr/bin/env python
"""Headline benchmark: MF-CIM spin-steps/s on BASELINE.json config 1.

Workload (one "step" of this script = one full pass of the hot path over the
batch): 64 seeded gen_instance(N=2000, alpha=0.5, a=0.1, nu=0.01) instances x
16 replicas, K1 gram build, 20 alternations (velo=19) x 1000 fused Euler
steps (dt 0.01, linear pump 0 -> 1.2) + damped-Jacobi refit (100 sweeps) +
scoring.  Inputs (A, y) are resident in HBM when the timed region starts;
the 1 GB gram (fp32) is larger than L2, so no flush is needed.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                  [--dtype f32|f64]

Multi-GPU (torchrun, one rank per GPU): every rank solves its own 64-instance
batch (seeds offset by rank) -- weak scaling, no data-path collective; the
step time is the max over ranks.  ``--impl reference`` times the CPU
restatement of the reference path (oracle/, matrix-free A^T(A w), no FMA,
one trajectory per host thread as the reference's run_jobs pool) on a
bounded sample of the same workload.
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


def ncu_traffic():
    """Per-launch DRAM traffic of the step kernel from the committed ncu capture."""
    p = os.path.join(ROOT, "profiles", "ncu_step_summary.json")
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


def ctx_nr(R, dtype):
    """Replica slots of a context: a power of two (>= 8 on the tensor-core path)."""
    p = 1
    while p < R:
        p *= 2
    return max(8, p) if dtype == "f32" else p


def kernel_label(N, NR, dtype):
    """The dominant kernel of the run (runtime.cu dispatch: cluster_ok / launch_gemv)."""
    if N <= 512 and NR <= (4 if dtype == "f64" else 8):
        t = "double" if dtype == "f64" else "float"
        return (f"cluster_loop_kernel<{t},{NR},BN> (whole 1000-step CIM call per launch, G "
                "register-resident, w over DSMEM; bound by the per-step FMA chain + DSMEM "
                "round trip, so the HBM fraction is an HBM-equivalent figure)")
    if dtype == "f32":
        return (f"sym_step_kernel<{NR},BN> + sym_update_kernel<{NR},BN> (one fused "
                "Euler step: upper-triangle gram tiles as fp16 hi/lo, each read once for G w "
                "and G^T w on tcgen05; achieved counts the stored triangle bytes one step must "
                "read, dense_equivalent the dense fp32 gram share of SURVEY 8(d))")
    return f"gemv_fused_kernel<double,{NR},BN> (fused Euler step, fp64 DFMA)"


def make_instances(rank, config=1, ws=1):
    """(instances, replicas, hyper-params, default dtype) of a BASELINE config.
    Config 1 is weak-scaled (each rank its own 64 instances); config 2's fixed
    1344-instance sweep is split into cost-balanced contiguous blocks."""
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
    return W.config1(rank, CFG["B"])


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


def cpu_sample(insts, nthreads, alt_limit=1, n_steps=None):
    """Bounded CPU sample: one trajectory per host thread, first alt_limit
    alternations (n_steps Euler steps each + refit + scoring), reference-literal
    coupling (A^T(A w), orchestrator.cpp:86-88)."""
    from oracle import oracle as O
    n_steps = n_steps or CFG["n_steps"]
    hp = O.baseline_params(velo=CFG["velo"], n_steps=n_steps)
    n = nthreads
    sel = [insts[k % len(insts)] for k in range(n)]
    oinst = [O.Instance(i.A, i.y, i.x_true, i.xi_true) for i in sel]
    seeds = np.array([O.mix_seed(i.seed, 1 + 3 * (k // len(insts)))
                      for k, i in enumerate(sel)], np.uint64)
    wall, _, _ = O.solve_batch_limited(oinst, seeds, hp, nthreads, alt_limit=alt_limit,
                                       backend=O.MFZ_BN, mode=O.LITERAL)
    spin_steps = n * insts[0].N * n_steps * alt_limit
    return spin_steps / wall, wall, n


def cpu_sample_steps(inst, nthreads, n_steps):
    """Config 4 CPU sample: nthreads trajectories x n_steps Euler steps of run_mfz
    with the reference's matrix-free A^T(A w) (no refit: its k x k gram alone is
    O(M k^2)).  One oracle problem per thread (its LITERAL scratch is per problem,
    A is shared read-only); only the steps are timed (ctypes releases the GIL)."""
    import threading
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


def run_reference(args, ws, rank):
    if rank != 0:
        return
    insts, _, _, _ = make_instances(0, args.config)
    nthreads = os.cpu_count() or 1
    vals, walls = [], []
    for k in range(args.warmup + args.steps):
        v, wall, n = cpu_sample(insts, nthreads)
        if k >= args.warmup:
            vals.append(v)
            walls.append(wall)
    v = statistics.median(vals)
    sample = (f"{nthreads} trajectories (1 per host thread) of config-1 instances, each 1 "
              f"alternation = {CFG['n_steps']} Euler steps + 100-sweep Jacobi refit + scoring, "
              "fp64 matrix-free A^T(A w) as orchestrator.cpp:86-88")
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": ws,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * statistics.median(walls),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded gen_instance, datagen.cpp:15-55)",
        "config": {"workload": WORKLOADS[args.config], "sample": "bounded CPU sample"},
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": nthreads, "kind": "port",
                         "sample": sample},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def run_ours(args, ws, rank, local):
    import paper_2405_00366_b200 as P
    from paper_2405_00366_b200 import _lib
    _lib.load()  # before torch: the system cuBLAS 12.9 (fp32-emulated gram GEMMs) wins
    import torch

    torch.cuda.set_device(local)
    dist = None
    if ws > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl")
    device_gen = args.device_gen and args.config == 4
    if device_gen:  # counter-based instance drawn on the GPU (a deviation)
        from paper_2405_00366_b200.workloads import config4 as _c4
        _, R, hp, wdtype = _c4(N=8)
        Nd = CFG.get("n4", 100_000)
        gen_params = [(0.5, 0.05, 0.01, 7)]
        Md, _ = P.gen_dims(Nd, 0.5, 0.05)
        insts = [P.Instance(np.zeros((Md, 0)), np.zeros(0), seed=7)]  # shape/seed stand-in
    else:
        insts, R, hp, wdtype = make_instances(rank, args.config, ws)
    if args.dtype is None:
        args.dtype = wdtype
    seeds = P.replica_seeds(insts, R, "mfz-bn")
    nalt = hp.velo + 1
    Bn, Nn = len(insts), (Nd if device_gen else insts[0].N)
    units = Bn * R * Nn * hp.n_steps * nalt  # spin-steps per rank per step
    # config 4 on several GPUs (or --shard): ONE instance split by gram tiles
    # across the ranks (tile-sharded contexts: replicated state, one NCCL
    # all-reduce per step) -- strong scaling, every rank counts 1/ws of it
    tile_sharded = args.config == 4 and (ws > 1 or args.shard)

    def make_ctx():
        if not tile_sharded:
            return P.Context(local, args.dtype)
        nid = [P.nccl_unique_id() if rank == 0 else None]
        if dist is not None:
            dist.broadcast_object_list(nid, src=0)
        return P.Context(local, args.dtype, shard=(ws, rank, nid[0]))

    if tile_sharded:
        units = units / ws
    ctx = make_ctx()

    def load_problems(cx):
        if device_gen:
            cx.set_generated_problems(Nd, gen_params)
        else:
            cx.set_problems(insts)

    t_gen = time.perf_counter()
    load_problems(ctx)
    torch.cuda.synchronize()
    gen_s = time.perf_counter() - t_gen

    def one_step():
        ctx.build_coupling()
        res = ctx.solve(R, "mfz-bn", hp, seeds)
        tm = ctx.timing()
        return res, tm

    for _ in range(args.warmup):
        one_step()

    def barrier():
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    dev_ms, step_ms_list, launches = [], [], 0
    gram_ms, cim_ms, refit_ms, score_ms = [], [], [], []
    barrier()
    with ClockSampler(local) as clocks:
        t0 = time.perf_counter()
        for _ in range(args.steps):
            res, tm = one_step()
            dev_ms.append(tm["gram_ms"] + tm["total_ms"])
            gram_ms.append(tm["gram_ms"])
            cim_ms.append(tm["cim_ms"])
            refit_ms.append(tm["refit_ms"])
            score_ms.append(tm["score_ms"])
            step_ms_list.append(tm["cim_ms"] / (nalt * hp.n_steps))
            launches += int(tm["step_launches"] + tm["refit_launches"] + tm["other_launches"]) + 2
        barrier()
        wall = time.perf_counter() - t0
    total_dev_ms = sum(dev_ms)
    if dist is not None:
        t = torch.tensor([total_dev_ms], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_dev_ms = float(t.item())
    ms_per_step = total_dev_ms / args.steps
    total_units = units
    if dist is not None:  # config 2 shards are uneven: sum what every rank processed
        t = torch.tensor([float(units)], device="cuda", dtype=torch.float64)
        dist.all_reduce(t)
        total_units = float(t.item())
    value = total_units / (ms_per_step * 1e-3)

    # roofline of the dominant kernel (the fused Euler step)
    es = 4 if args.dtype == "f32" else 8
    dense_bytes = Bn * Nn * Nn * es  # the dense G share, s*N/R per spin-step
    step_bytes = dense_bytes
    if args.dtype == "f32" and not (Nn <= 512 and ctx_nr(R, args.dtype) <= 8):
        # symmetric-tile path: the upper-triangle 128x128 tiles as fp16 hi|lo
        # (4 bytes per stored entry), read once per step for G w and G^T w
        nrb = (Nn + 127) // 128
        step_bytes = Bn * (nrb * (nrb + 1) // 2) * 128 * 128 * 4
    step_s = statistics.median(step_ms_list) * 1e-3
    peak, peak_kind = measured_peaks()
    if tile_sharded:  # per GPU: each rank streams its share of the gram tiles
        step_bytes = step_bytes / ws
        dense_bytes = dense_bytes / ws
    achieved = step_bytes / step_s / 1e9

    # e2e: public API with HOST buffers, H2D of the instances and D2H of results inside
    e2e_val, h2d, d2h = None, 0, 0
    if not args.no_e2e:
        ctx2 = make_ctx()

        def e2e_once():
            load_problems(ctx2)
            ctx2.build_coupling()
            out = ctx2.solve(R, "mfz-bn", hp, seeds)
            torch.cuda.synchronize()
            return out

        e2e_once()  # untimed: first-use allocations and graph capture of the context
        barrier()
        e2e_times = []
        for _ in range(max(1, min(args.steps, 3))):
            t1 = time.perf_counter()
            r2 = e2e_once()
            e2e_times.append(time.perf_counter() - t1)
            print(f"e2e run {e2e_times[-1]:.3f}s", file=sys.stderr)
        ctx2.close()
        e2e_s = statistics.median(e2e_times)
        if dist is not None:
            t = torch.tensor([e2e_s], device="cuda", dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e2e_s = float(t.item())
        e2e_val = total_units / e2e_s
        h2d = 0 if device_gen else sum(i.A.nbytes + i.y.nbytes + i.x_true.nbytes +
                                       i.xi_true.nbytes for i in insts)
        h2d += Bn * R * Nn * 8 * nalt  # host-drawn c0 streams
        d2h = r2["R"].nbytes + r2["sigma"].nbytes + r2["history"].nbytes

    # the dominant kernel alone: a short eager run with CUDA events around every
    # step-mode launch of the tile kernel on its stream (outside the timed region;
    # the step-level roofline above is the in-region figure)
    dom = None
    if args.dtype == "f32" and not (Nn <= 512) and not tile_sharded:
        ctx.set_option("use_graphs", 0)
        ctx.set_option("kernel_timing", 1)
        ctx.solve(R, "mfz-bn", P.baseline_params(velo=1, n_steps=100), seeds)
        tk = ctx.timing()
        ctx.set_option("kernel_timing", 0)
        ctx.set_option("use_graphs", 1)
        if tk["tile_kernel_launches"] > 0:
            t_tile = tk["tile_kernel_ms"] / tk["tile_kernel_launches"] * 1e-3
            dom = {"kernel": f"sym_step_kernel<{ctx_nr(R, args.dtype)},BN>",
                   "avg_us": t_tile * 1e6, "launches": int(tk["tile_kernel_launches"]),
                   "bytes_per_launch": step_bytes, "achieved": step_bytes / t_tile / 1e9,
                   "peak": peak, "unit": "GB/s", "frac": step_bytes / t_tile / 1e9 / peak,
                   "share_of_step": t_tile / step_s,
                   "how": ("eager run of 2 x 100 steps after the timed region, CUDA events on "
                           "the launch stream around each launch (serialised: the kernel "
                           "timed alone, burst peak)")}

    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu and not device_gen:
        nthreads = os.cpu_count() or 1
        if args.config == 4:
            cs = 2
            v, wall_c, n = cpu_sample_steps(insts[0], min(nthreads, 8), cs)
            sample = (f"{n} trajectories (1/host thread) x {cs} Euler steps of run_mfz, fp64 "
                      f"A^T(A w) restatement, no refit, {wall_c:.1f}s wall")
        else:
            cs = 100 if args.config == 3 else hp.n_steps  # config 3: 100-step sample
            v, wall_c, n = cpu_sample(insts, nthreads, n_steps=cs)
            sample = (f"{n} trajectories (1/host thread) x 1 alternation x {cs} Euler steps "
                      f"+ refit, fp64 A^T(A w) restatement, {wall_c:.1f}s wall")
        cpu = {"value": v, "unit": UNIT, "cores": nthreads, "kind": "port", "sample": sample}
    ctx.close()
    fp64 = None
    if args.dtype == "f32" and not args.no_fp64 and args.config == 1:
        c64 = P.Context(local, "f64")
        c64.set_problems(insts)
        c64.build_coupling()
        c64.solve(R, "mfz-bn", hp, seeds)  # warm-up
        barrier()
        c64.build_coupling()
        c64.solve(R, "mfz-bn", hp, seeds)
        t64 = c64.timing()
        c64.close()
        ms64 = t64["gram_ms"] + t64["total_ms"]
        st64 = t64["cim_ms"] / (nalt * hp.n_steps) * 1e-3
        ach64 = 2 * dense_bytes / st64 / 1e9 if args.dtype == "f32" else None  # dense fp64 G
        fp64 = {"value": total_units / (ms64 * 1e-3), "unit": UNIT, "ms_per_step": ms64,
                "steps": 1, "warmup": 1,
                "note": "fp64 path (bitwise-parity mode, CUDA-core DFMA contraction)",
                "roofline": {"bound": "hbm", "achieved": ach64, "peak": peak, "unit": "GB/s",
                             "frac": ach64 / peak}}
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": "strong" if args.config == 2 or tile_sharded else "weak",
            "vs_baseline": None,
            "dtype": args.dtype,
            "data": ("synthetic, generated on the GPU from counter-based Philox streams "
                     "(documented deviation: not the reference's mt19937_64 instance)"
                     if device_gen else "synthetic (seeded gen_instance, datagen.cpp:15-55)"),
            "config": {"workload": (WORKLOADS[args.config] if args.config != 4 or args.n4 == 100_000
                                    else WORKLOADS[4].replace("N=100000 M=50000 K=5000",
                                                              f"N={Nn} (reduced)")),
                       "per_rank_instances": Bn, "replicas": R,
                       "parallelism": (f"tile-sharded gram x{ws} (replicated state, one NCCL "
                                       "all-reduce per step)" if tile_sharded else
                                       f"instance shards x{ws}"),
                       "step": "gram build + full alternating solve",
                       "l2": ("inputs larger than L2 (gram %.2f GB per step)" % (step_bytes / 1e9)
                              if step_bytes > 126e6 else "gram fits in L2 (no flush)")},
            "instances_per_s": (Bn if tile_sharded else total_units / units * Bn) / (ms_per_step * 1e-3),
            "problem_load_s": gen_s,
            "breakdown_ms": {"gram": statistics.median(gram_ms), "cim": statistics.median(cim_ms),
                             "refit": statistics.median(refit_ms),
                             "score": statistics.median(score_ms)},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak,
                         "traffic": ncu_traffic() if args.config == 1 and args.dtype == "f32" else None,
                         "traffic_note": ("ncu dram read+write of the three kernels of one step "
                                          "(profiles/ncu_step_summary.json)"
                                          if args.config == 1 and args.dtype == "f32" else None),
                         "kernel": kernel_label(Nn, ctx_nr(R, args.dtype), args.dtype),
                         "bytes_per_launch": step_bytes, "peak_kind": peak_kind,
                         "dominant_kernel": dom,
                         "dense_equivalent": {"bytes_per_launch": dense_bytes,
                                              "achieved": dense_bytes / step_s / 1e9}},
            "e2e": None if e2e_val is None else {
                "value": e2e_val, "unit": UNIT, "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h},
            "gpu_launches": launches,
            "clocks": clocks.summary(),
            "wall_s": wall,
        }
        if cpu is not None:
            line["cpu_baseline"] = cpu
        if fp64 is not None:
            line["fp64"] = fp64
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
            "roofline": {"bound": "latency",
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


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--dtype", default=None, choices=["f32", "f64"],
                    help="default: the config's (f32 for 1-3, f64 for 0)")
    ap.add_argument("--config", type=int, default=1, choices=[0, 1, 2, 3, 4])
    ap.add_argument("--n4", type=int, default=100_000, help="config 4 size (N)")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-fp64", action="store_true", help="skip the fp64 secondary line")
    ap.add_argument("--device-gen", action="store_true",
                    help="config 4: generate the instance on the GPU (counter-based deviation)")
    ap.add_argument("--shard", action="store_true",
                    help="config 4: use the tile-sharded context even on one GPU")
    ap.add_argument("--mri", action="store_true",
                    help="the reference's matrix-free MRI chain at config-3 size (run_mri)")
    args = ap.parse_args()
    CFG["n4"] = args.n4
    ws, rank, local = dist_env()
    if args.mri and args.impl == "ours":
        run_mri(args, ws, rank, local)
    elif args.impl == "reference":
        run_reference(args, ws, rank)
    else:
        run_ours(args, ws, rank, local)


if __name__ == "__main__":
    main()
