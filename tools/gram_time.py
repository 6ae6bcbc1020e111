"""Time of the large-N tcgen05 gram build (gram_tc_kernel) on device-generated
instances, vs the persistent CTAs used (option sched_ctas limits them: is the build
bound by a shared resource -- L2 / HBM -- or by the SM's own pipeline?).
Run on the B200 box:  python tools/gram_time.py [N] [ctas,ctas,...]"""
from __future__ import annotations
import json, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2405_00366_b200 as P  # noqa: E402


def main():
    N = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
    ctas = [int(x) for x in sys.argv[2].split(",")] if len(sys.argv) > 2 else [148, 111, 74]
    out = {}
    for n in ctas:
        with P.Context(0, "f32") as ctx:
            ctx.set_option("sched_ctas", n)
            ctx.set_generated_problems(N, [(0.5, 0.05, 0.01, 7)])
            best = 1e30
            for _ in range(2):
                ctx.build_coupling()
                best = min(best, ctx.timing()["gram_ms"])
        M, _ = P.gen_dims(N, 0.5, 0.05)
        nrb = (N + 127) // 128
        steps = nrb * (nrb + 1) // 2 * ((M + 31) // 32)
        out[n] = {"gram_ms": best, "us_per_chunk_step_per_cta": 1e3 * best * n / steps,
                  "pflops_split_mma": 3 * 2.0 * 128 * 128 * 32 * steps / (best * 1e-3) / 1e15}
        print(N, M, n, json.dumps(out[n]), flush=True)
    json.dump(out, open(os.path.join(ROOT, "gpurun_out", f"gram_time_{N}.json"), "w"), indent=1)


if __name__ == "__main__":
    main()
