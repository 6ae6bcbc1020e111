"""Per-chunk pipeline stamps of gram_tc_kernel's CTA 0 (option "timeline"): where
does a k-chunk's time go?  Run on the B200 box: python tools/gram_pipeline.py [N]"""
from __future__ import annotations
import json, os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2405_00366_b200 as P  # noqa: E402

def main():
    N = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
    with P.Context(0, "f32") as ctx:
        ctx.set_option("timeline", 1)
        ctx.set_generated_problems(N, [(0.5, 0.05, 0.01, 7)])
        ctx.build_coupling()
        ctx.build_coupling()
        tl = ctx.timeline().astype(np.int64)
    a = tl[8192:8192 + 128]
    e = tl[8192 + 128:8192 + 256]
    t0 = a[0, 0]
    a = (a - t0) / 1e3
    e = (e - t0) / 1e3
    print("it  acc_free  landed  issued | stage_free(prod) | epi_ready epi_released")
    for t in range(40, 72):
        print(f"{t:3d} {a[t,0]:8.2f} {a[t,1]:8.2f} {a[t,2]:8.2f} | {a[t,3]:8.2f} | {e[t,0]:8.2f} {e[t,1]:8.2f}")
    s = slice(16, 120)
    d = {"per_chunk_us": float((a[119, 2] - a[16, 2]) / 103),
         "wait_acc_us": float(np.mean(a[s, 0][1:] - a[s, 2][:-1])),
         "wait_landed_us": float(np.mean(a[s, 1] - a[s, 0])),
         "issue_us": float(np.mean(a[s, 2] - a[s, 1])),
         "issue_to_epi_ready_us": float(np.mean(e[s, 0] - a[s, 2])),
         "epi_read_us": float(np.mean(e[s, 1] - e[s, 0]))}
    print(json.dumps(d, indent=1))
    json.dump(d, open(os.path.join(ROOT, "gpurun_out", "gram_pipeline.json"), "w"), indent=1)

if __name__ == "__main__":
    main()
