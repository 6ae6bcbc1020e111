"""Random shapes through the low-level C-ABI calls of an fp64 context (and the fp32 unit
tolerances on the same problems) -- one fused step
(cimcs_mfz_step), a whole CIM call (cimcs_run_cim), the refit (cimcs_cdp_minimize, Jacobi
and CG) and the scorer (cimcs_score) -- bitwise against the oracle in the context's
canonical order (scalars of the scorer 1e-12 relative).  Run on the B200 box."""
from __future__ import annotations
import math, os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2405_00366_b200 as P  # noqa: E402
from oracle import oracle as O  # noqa: E402  (the checker)


def run(cases, seed, quiet=False):
    rng = np.random.default_rng(seed)
    bad = 0
    for ci in range(cases):
        N = int(rng.choice([33, 200, 512, 513, 577, 640, 1100, 1537, 2049]))
        B = int(rng.choice([1, 2, 5, 11]))
        R = int(rng.choice([1, 3, 8, 16]))
        insts = [O.gen_instance(N, float(rng.uniform(0.3, 0.9)), float(rng.uniform(0.05, 0.4)), 0.01,
                                1000 * ci + s) for s in range(B)]
        backend = str(rng.choice(["mfz-bn", "mfz-cn"]))
        be = O.MFZ_BN if backend == "mfz-bn" else O.MFZ_CN
        tag = f"case {ci}: N={N} B={B} R={R} {backend}"
        msgs = []
        try:
            with P.Context(0, "f64") as ctx:
                ctx.set_problems(insts)
                ctx.build_coupling()
                order = ctx.canon_order()
                probs = [O.Problem(i, O.CANON, *order) for i in insts]
                b, r = B - 1, R - 1
                # one step
                Rs = rng.normal(size=(B, R, N)); c = rng.normal(scale=0.5, size=(B, R, N))
                e = np.abs(rng.normal(size=(B, R, N))) + 0.1
                hp, ghp = O.baseline_params(), P.baseline_params()
                out = ctx.mfz_step(R, backend, ghp, 0.37, 0.83, Rs, c, e)
                h = (probs[b].local_field_bn(Rs[b, r], (c[b, r] > 0).astype(np.int32), hp.tau)
                     if backend == "mfz-bn" else probs[b].local_field_cn(Rs[b, r], c[b, r], hp.tau))
                co, eo = O.mfz_step(c[b, r], e[b, r], 0.83, hp, 0.37, Rs[b, r], h)
                ok = (np.array_equal(out["h"][b, r], h) and np.array_equal(out["c"][b, r], co)
                      and np.array_equal(out["e"][b, r], eo))
                msgs.append("step " + ("OK" if ok else "BAD")); bad += not ok
                # CIM call
                ns = int(rng.integers(10, 90))
                seeds = [[O.mix_seed(i.seed, 1 + 3 * q) for q in range(R)] for i in insts]
                c0 = np.zeros((B, R, N))
                for bb in range(B):
                    for q in range(R):
                        g = O.Rng(seeds[bb][q])
                        c0[bb, q] = [0.01 * g.gauss() for _ in range(N)]
                Rh = np.stack([np.stack([p.hz] * R) for p in probs])
                out = ctx.run_cim(R, backend, P.baseline_params(n_steps=ns), 0.5, Rh, c0)
                ref = probs[b].run_mfz(Rh[b, r], O.baseline_params(n_steps=ns), 0.5, be,
                                       O.Rng(seeds[b][r]))
                ok = (np.array_equal(out["c"][b, r], ref["c"]) and np.array_equal(out["e"][b, r], ref["e"])
                      and np.array_equal(out["sigma"][b, r], ref["sigma"]) and out["min_e"][b, r] == ref["min_e"])
                msgs.append("cim " + ("OK" if ok else "BAD")); bad += not ok
                # refit, both methods
                sigma = (rng.random((B, R, N)) < float(rng.uniform(0.05, 0.9))).astype(np.int32)
                Rp = rng.normal(size=(B, R, N))
                for method, name in ((O.CDP_JACOBI, "jacobi"), (O.CDP_CG, "cg")):
                    got = ctx.refit(R, sigma, Rp, P.HyperParams(), cdp=name)
                    ref = probs[b].cdp(sigma[b, r], Rp[b, r], method, O.HyperParams())
                    ok = np.array_equal(got[b, r], ref)
                    msgs.append(name + (" OK" if ok else " BAD")); bad += not ok
                # score
                out = ctx.score(R, Rp, sigma, 0.05)
                obj = probs[b].objective_at(Rp[b, r], sigma[b, r], 0.05)
                rm = O.rmse(Rp[b, r], sigma[b, r], insts[b].x_true, insts[b].xi_true)
                ok = (math.isclose(out["objective"][b, r], obj, rel_tol=1e-12)
                      and math.isclose(out["rmse"][b, r], rm, rel_tol=1e-12)
                      and out["hamming"][b, r] == O.hamming_loss(sigma[b, r], insts[b].xi_true))
                msgs.append("score " + ("OK" if ok else "BAD")); bad += not ok
            # the fp32 path on the same problem: field within 2e-5 of its scale, one Jacobi
            # refit within 1e-4, score within 1e-4 (the fp32 unit tolerances)
            with P.Context(0, "f32") as ctx:
                ctx.set_problems(insts)
                ctx.build_coupling()
                pc = [O.Problem(i, O.CANON) for i in (insts[b],)][0]
                out = ctx.mfz_step(R, backend, ghp, 0.37, 0.83, Rs, c, e)
                h = (pc.local_field_bn(Rs[b, r], (c[b, r] > 0).astype(np.int32), hp.tau)
                     if backend == "mfz-bn" else pc.local_field_cn(Rs[b, r], c[b, r], hp.tau))
                eh = float(np.max(np.abs(out["h"][b, r] - h)) / np.max(np.abs(h)))
                got = ctx.refit(R, sigma, Rp, P.HyperParams(), cdp="jacobi")
                ref = pc.cdp(sigma[b, r], Rp[b, r], O.CDP_JACOBI, O.HyperParams())
                er = float(np.max(np.abs(got[b, r] - ref)) / max(np.max(np.abs(ref)), 1e-30))
                sc = ctx.score(R, Rp, sigma, 0.05)
                es = abs(sc["objective"][b, r] - obj) / max(abs(obj), 1e-30)
                ok = eh < 2e-5 and er < 1e-4 and es < 1e-4
                msgs.append(f"f32 h {eh:.1e} refit {er:.1e} obj {es:.1e} " + ("OK" if ok else "BAD"))
                bad += not ok
        except Exception as ex:  # noqa: BLE001
            msgs.append("ERROR " + str(ex)[:140]); bad += 1
        if not quiet or any("OK" not in m for m in msgs):
            print(tag, "->", ", ".join(msgs), flush=True)
    return bad


if __name__ == "__main__":
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 20
    bad = run(n, int(sys.argv[2]) if len(sys.argv) > 2 else 0)
    print("bad:", bad)
    sys.exit(1 if bad else 0)
