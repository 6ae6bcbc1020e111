"""Randomised shape check of the fp64 path against the oracle (bitwise) and of the
fp32 path against the fp64 path (no errors, finite, close first supports): odd N, small
and larger batches, replica counts that pad, both MFZ backends, Jacobi and CG refits,
Positive-P.  Run on the B200 box: python tools/shape_fuzz.py [cases] [seed]"""
from __future__ import annotations
import os, sys, time
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2405_00366_b200 as P  # noqa: E402
from oracle import oracle as O  # noqa: E402  (the checker)


def run(cases, seed, quiet=False):
    """Returns the number of bad cases (fp64 mismatch, fp32 non-finite, or an error)."""
    rng = np.random.default_rng(seed)
    bad = 0
    for ci in range(cases):
        N = int(rng.choice([33, 97, 200, 500, 512, 513, 520, 577, 640, 1025, 1100, 1537, 2000, 2049,
                            3000]))
        B = int(rng.choice([1, 2, 5, 12, 33]))
        R = int(rng.choice([1, 3, 8, 16]))
        backend = str(rng.choice(["mfz-bn", "mfz-cn", "pp"]))
        cdp = str(rng.choice(["jacobi", "cg"])) if backend != "pp" else "jacobi"
        alpha, a = float(rng.uniform(0.25, 0.95)), float(rng.uniform(0.02, 0.6))
        velo, n_steps = int(rng.integers(1, 5)), int(rng.integers(20, 160))
        track_best = bool(rng.integers(0, 2)) and backend != "pp"
        # context variants: plain, world-1 sharded (tile sharding in fp32, row sharding in
        # fp64: same results as plain), option toggles that must not change fp64 bits
        variant = str(rng.choice(["plain", "plain", "sharded", "no_graphs", "no_cluster", "no_pdl"]))
        insts = [O.gen_instance(N, alpha, a, 0.01, 1000 * ci + s) for s in range(B)]
        be = O.BACKENDS[backend]
        seeds = np.array([[O.mix_seed(i.seed, be + 3 * r) for r in range(R)] for i in insts],
                         np.uint64)
        kw = dict(velo=velo, n_steps=n_steps, g2=0.01) if backend == "pp" else dict(velo=velo, n_steps=n_steps)
        ghp = P.HyperParams(**kw) if backend == "pp" else P.baseline_params(**kw)
        ohp = O.HyperParams(**kw) if backend == "pp" else O.baseline_params(**kw)
        tag = (f"case {ci}: N={N} B={B} R={R} {backend} {cdp} velo={velo} steps={n_steps} "
               f"best={int(track_best)} {variant}")
        t0 = time.time()
        try:
            def make(dt):
                sharded = variant == "sharded" and backend != "pp"
                ctx = P.Context(0, dt, shard=(1, 0, P.cimcs.nccl_unique_id()) if sharded else None)
                if variant == "no_graphs":
                    ctx.set_option("use_graphs", 0)
                if variant == "no_cluster":
                    ctx.set_option("cluster_loop", 0)
                if variant == "no_pdl":
                    ctx.set_option("pdl", 0)
                return ctx
            with make("f64") as ctx:
                ctx.set_problems(insts)
                ctx.build_coupling()
                order = ctx.canon_order()
                r64 = ctx.solve(R, backend, ghp, seeds, cdp=cdp, track_best=track_best)
            ok = True
            for (b, r) in {(0, 0), (B - 1, R - 1)}:
                ref = O.Problem(insts[b], O.CANON, *order).alternating_minimize(
                    be, ohp, O.Rng(int(seeds[b, r])), cdp=(O.CDP_CG if cdp == "cg" else O.CDP_JACOBI),
                    track_best=track_best)
                if ref.get("failed"):
                    ok &= bool(r64["fail_alt"][b, r] == ref["fail_alternation"])
                else:
                    ok &= bool(np.array_equal(r64["R"][b, r], ref["R"]) and
                               np.array_equal(r64["sigma"][b, r], ref["sigma"]))
            msg = "fp64 bitwise " + ("OK" if ok else "MISMATCH")
            if not ok:
                bad += 1
            with make("f32") as ctx:
                ctx.set_problems(insts)
                ctx.build_coupling()
                r32 = ctx.solve(R, backend, ghp, seeds, cdp=cdp, track_best=track_best)
            fin = bool(np.all(np.isfinite(r32["R"])))
            same = float(np.mean(np.all(r32["sigma"] == r64["sigma"], axis=2)))
            msg += f" | fp32 finite {fin} same-support {same:.2f}"
            if not fin:
                bad += 1
        except Exception as e:  # noqa: BLE001
            msg = "ERROR " + str(e)[:160]
            bad += 1
        if not quiet or "OK |" not in msg:
            print(tag, "->", msg, f"({time.time() - t0:.1f}s)", flush=True)
    return bad


def main():
    cases = int(sys.argv[1]) if len(sys.argv) > 1 else 16
    bad = run(cases, int(sys.argv[2]) if len(sys.argv) > 2 else 0)
    print("bad cases:", bad)
    return 1 if bad else 0


if __name__ == "__main__":
    sys.exit(main())
