"""Context-reuse check: ONE fp64 context (and one fp32 context) is driven through a random
sequence of set_problems / build_coupling / solve / run_cim / refit calls whose shapes (N, B,
per-instance M), replica counts, schedules and backends change from call to call -- cached
graphs, item schedules, state and pump buffers must follow.  Every fp64 solve is compared
bitwise with the oracle; fp32 results must be finite.
Run on the B200 box: python tools/reuse_fuzz.py [sequences] [seed]"""
from __future__ import annotations
import os, sys, time
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2405_00366_b200 as P  # noqa: E402
from oracle import oracle as O  # noqa: E402  (the checker)


def run(nseq, seed, quiet=False):
    rng = np.random.default_rng(seed)
    bad = 0
    for si in range(nseq):
        ctx64, ctx32 = P.Context(0, "f64"), P.Context(0, "f32")
        log = []
        try:
            insts = None
            for step in range(int(rng.integers(3, 7))):
                if insts is None or rng.random() < 0.5:  # new problem set, per-instance M differs
                    N = int(rng.choice([97, 500, 513, 640, 1100, 2000]))
                    B = int(rng.choice([1, 2, 5, 9]))
                    insts = [O.gen_instance(N, float(rng.uniform(0.3, 0.9)), float(rng.uniform(0.05, 0.3)),
                                            0.01, 100 * si + 10 * step + s) for s in range(B)]
                    for c in (ctx64, ctx32):
                        c.set_problems(insts)
                        c.build_coupling()
                R = int(rng.choice([1, 3, 8, 16]))
                backend = str(rng.choice(["mfz-bn", "mfz-cn", "pp"]))
                cdp = str(rng.choice(["jacobi", "cg"])) if backend != "pp" else "jacobi"
                velo, n_steps = int(rng.integers(1, 4)), int(rng.integers(20, 120))
                be = O.BACKENDS[backend]
                seeds = np.array([[O.mix_seed(i.seed, be + 3 * r) for r in range(R)] for i in insts],
                                 np.uint64)
                kw = dict(velo=velo, n_steps=n_steps)
                ghp = P.HyperParams(g2=0.01, **kw) if backend == "pp" else P.baseline_params(**kw)
                ohp = O.HyperParams(g2=0.01, **kw) if backend == "pp" else O.baseline_params(**kw)
                log.append(f"N={insts[0].N} B={len(insts)} R={R} {backend} {cdp} {velo}x{n_steps}")
                r64 = ctx64.solve(R, backend, ghp, seeds, cdp=cdp)
                order = ctx64.canon_order()
                b, r = len(insts) - 1, R - 1
                ref = O.Problem(insts[b], O.CANON, *order).alternating_minimize(
                    be, ohp, O.Rng(int(seeds[b, r])), cdp=(O.CDP_CG if cdp == "cg" else O.CDP_JACOBI))
                ok = (bool(r64["fail_alt"][b, r] == ref["fail_alternation"]) if ref.get("failed") else
                      bool(np.array_equal(r64["R"][b, r], ref["R"]) and
                           np.array_equal(r64["sigma"][b, r], ref["sigma"])))
                r32 = ctx32.solve(R, backend, ghp, seeds, cdp=cdp)
                fin = bool(np.all(np.isfinite(r32["R"])))
                log[-1] += " OK" if ok and fin else f" BAD(fp64={ok}, fp32 finite={fin})"
                if not (ok and fin):
                    bad += 1
        except Exception as e:  # noqa: BLE001
            log.append("ERROR " + str(e)[:140])
            bad += 1
        finally:
            try:
                ctx64.close()
                ctx32.close()
            except Exception:  # noqa: BLE001
                pass
        if not quiet or any("OK" not in x for x in log):
            print(f"sequence {si}: " + " | ".join(log), flush=True)
    return bad


if __name__ == "__main__":
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 10
    bad = run(n, int(sys.argv[2]) if len(sys.argv) > 2 else 0)
    print("bad:", bad)
    sys.exit(1 if bad else 0)
