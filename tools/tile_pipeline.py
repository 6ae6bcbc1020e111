"""Per-tile pipeline stamps of tile CTA 0 (option "timeline") for the last Euler
step of a config-1 CIM call: where does a tile's 1.6 us go?  Run on the B200 box."""
from __future__ import annotations
import json, os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2405_00366_b200 as P  # noqa: E402
from paper_2405_00366_b200 import workloads as W  # noqa: E402

def main():
    insts, R, hp, _ = W.config1(0, 64)
    hp = P.baseline_params(velo=1, n_steps=300)
    B, N = len(insts), insts[0].N
    rng = np.random.default_rng(0)
    Rs = np.abs(rng.normal(size=(B, R, N))) * 0.1
    c0 = rng.normal(scale=1e-2, size=(B, R, N))
    with P.Context(0, "f32") as ctx:
        ctx.set_option("timeline", 1)
        ctx.set_problems(insts)
        ctx.build_coupling()
        for _ in range(2):
            ctx.run_cim(R, "mfz-bn", hp, 0.5, Rs, c0)
        tl = ctx.timeline().astype(np.int64)
    a = tl[8192:8192 + 128]
    e = tl[8192 + 128:8192 + 256]
    n = int((a[:, 1] > 0).sum())
    t0 = tl[0, 0]
    a = (a[:n] - t0) / 1e3
    e = (e[:n] - t0) / 1e3
    print("tile  acc_free  landed  issued | refill_issued | epi_acc_ready  epi_released")
    for t in range(n):
        print(f"{t:3d}  {a[t,0]:8.2f} {a[t,1]:8.2f} {a[t,2]:8.2f} | {a[t,3]:8.2f} | {e[t,0]:8.2f} {e[t,1]:8.2f}")
    d = {
        "tiles": n,
        "per_tile_us": float((a[-1, 2] - a[0, 2]) / (n - 1)),
        "wait_acc_us_mean": float(np.mean(np.maximum(a[2:, 0] - a[1:-1, 2], 0))),
        "wait_landed_us_mean": float(np.mean(a[2:, 1] - a[2:, 0])),
        "issue_us_mean": float(np.mean(a[2:, 2] - a[2:, 1])),
        "issue_to_acc_ready_us_mean": float(np.mean(e[2:, 0] - a[2:, 2])),
        "acc_read_us_mean": float(np.mean(e[2:, 1] - e[2:, 0])),
        "refill_to_landed_us_mean": float(np.mean(a[4:, 1] - a[4:, 3])),
    }
    print(json.dumps(d, indent=1))
    json.dump(d, open(os.path.join(ROOT, "gpurun_out", "tile_pipeline.json"), "w"), indent=1)

if __name__ == "__main__":
    main()
