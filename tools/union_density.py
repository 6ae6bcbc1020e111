"""Fraction of spins j with sigma_j = 1 in ANY of R replicas, per Euler step
(BN mode), on a config-1 instance: decides whether sigma-sparse skipping of
G rows pays.  Oracle, CPU."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from oracle import oracle as O  # noqa: E402

inst = O.gen_instance(2000, 0.5, 0.1, 0.01, 1)
hp = O.baseline_params()
p = O.Problem(inst, O.EXPLICIT)
R = 16
base = p.alternating_minimize(O.MFZ_BN, hp, O.Rng(O.mix_seed(1, 1)), keep=True)
for alt in (0, 5, 10, 19):
    Rv = p.hz if alt == 0 else base["hist_R"][alt - 1]
    eta = O.eta_schedule(alt, hp.eta_init, hp.eta_end, hp.velo)
    ups = []
    for r in range(R):
        tr = p.run_mfz(Rv, hp, eta, O.MFZ_BN, O.Rng(1000 + r), trace_mode=2)
        ups.append(tr["trace_c"][:-1] > 0)  # sigma used at each step
    U = np.any(np.stack(ups), axis=0)      # steps x N
    dens = U.mean(axis=1)
    # 4-spin K-group granularity (the tensor-core operand unit)
    Ug = U.reshape(U.shape[0], -1, 4).any(axis=2).mean(axis=1)
    print(f"alt {alt}: union density mean {dens.mean():.3f} (first100 {dens[:100].mean():.3f}, "
          f"last500 {dens[500:].mean():.3f}); 4-group density {Ug.mean():.3f}; "
          f"per-replica {np.mean([u.mean() for u in ups]):.3f}")
