"""One config-0 solve (fp64, N=500, 1 replica): the driver for ncu captures of
the small-N cluster loop kernel."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_2405_00366_b200 as P
from paper_2405_00366_b200 import workloads as W

insts, R, hp, dtype = W.config0()
velo = int(sys.argv[1]) if len(sys.argv) > 1 else 1
hp.velo = velo
ctx = P.Context(0, dtype)
ctx.set_problems(insts)
ctx.build_coupling()
res = ctx.solve(R, "mfz-bn", hp, P.replica_seeds(insts, R, "mfz-bn"))
t = ctx.timing()
print("cim_ms", t["cim_ms"], "refit_ms", t["refit_ms"], "per step us",
      1e3 * t["cim_ms"] / ((velo + 1) * hp.n_steps))
ctx.close()
