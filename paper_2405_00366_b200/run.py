"""Batch runner over instance bundles: the GPU counterpart of ``cimcs run
--load DIR --out DIR`` (tools/main.cpp:387-503).  Loads every bundle under
--load (sorted by seed), solves them as ONE batch on the B200 (B instances x R
replicas; replica 0 uses the reference's own solver seed mix_seed(seed,
backend), main.cpp:423), and writes summary.csv / history_<backend>.csv /
failures.csv with the reference's column contract.  With R > 1 the row of an
instance reports its best replica (minimum final objective)."""
from __future__ import annotations

import argparse
import sys

import numpy as np

from . import io as IO
from .cimcs import BACKENDS, HyperParams, baseline_params, replica_seeds, solve_batch, trial_dict


def run(load_dir: str, out_dir: str, backend: str = "mfz-bn", replicas: int = 1,
        dtype: str = "f64", params: HyperParams | None = None, device: int = 0) -> int:
    insts = IO.load_bundles(load_dir)
    if len({i.N for i in insts}) != 1:
        raise SystemExit("all bundles of one batch must share N")
    hp = params or HyperParams()
    seeds = replica_seeds(insts, replicas, backend)
    res = solve_batch(insts, replicas, backend, hp, seeds, dtype=dtype, device=device)
    trials = []
    for b in range(len(insts)):
        ts = [trial_dict(res, b, r, hp.n_steps) for r in range(replicas)]
        ok = [t for t in ts if not t["failed"]]
        best = min(ok, key=lambda t: t["history"][-1]["hamiltonian"]) if ok else ts[0]
        trials.append(best)
    cfg = IO.hex64(IO.fnv1a64(repr(sorted(vars(hp).items())) + backend + str(replicas)))
    return IO.write_run_tables(out_dir, insts, trials, backend, cfg)


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(description=__doc__)
    ap.add_argument("--load", required=True)
    ap.add_argument("--out", required=True)
    ap.add_argument("--backend", default="mfz-bn", choices=sorted(BACKENDS))
    ap.add_argument("--replicas", type=int, default=1)
    ap.add_argument("--dtype", default="f64", choices=("f32", "f64"))
    ap.add_argument("--baseline", action="store_true",
                    help="BASELINE.json schedule (linear pump 0->1.2, 20 x 1000 steps)")
    a = ap.parse_args(argv)
    hp = baseline_params() if a.baseline else HyperParams()
    failures = run(a.load, a.out, a.backend, a.replicas, a.dtype, hp)
    print(f"ran bundles under {a.load} -> {a.out} ({failures} failed)")
    return 0


if __name__ == "__main__":
    sys.exit(main())
