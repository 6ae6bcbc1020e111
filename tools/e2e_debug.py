"""Debug: config-2 instances loaded into two live contexts; report instances
whose diag(G) differs between them (bench e2e failure, r01h)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2405_00366_b200 as P  # noqa: E402
from paper_2405_00366_b200 import workloads as W  # noqa: E402

insts, R, hp, dt = W.config2()
print("B", len(insts), "M range", min(i.M for i in insts), max(i.M for i in insts), flush=True)
ctxs = []
for k in range(2):
    t = time.time()
    c = P.Context(0, "f32")
    c.set_problems(insts)
    c.build_coupling()
    ctxs.append(c)
    D = np.array([c.get_coupling(b, gram=False)[2] for b in range(len(insts))])
    zero = np.where(~(np.abs(D).max(axis=1) > 0))[0]
    print("ctx", k, "build s", round(time.time() - t, 1), "instances with zero/NaN D:", zero[:20], len(zero), flush=True)
    if k == 1:
        D0 = np.array([ctxs[0].get_coupling(b, gram=False)[2] for b in range(len(insts))])
        diff = np.where(np.any(D != D0, axis=1))[0]
        print("instances whose D differs between contexts:", diff[:20], len(diff), flush=True)
        ref = np.array([(np.asarray(i.A) ** 2).sum(axis=0) for i in insts[:4]])
        print("host D check (first 4):", np.max(np.abs(D[:4] - ref) / ref.max()), flush=True)
