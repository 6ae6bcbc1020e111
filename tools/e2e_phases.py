import sys, time
sys.path.insert(0, '.')
import paper_2405_00366_b200 as P
from paper_2405_00366_b200 import workloads as W
insts, R, hp, dt = W.config1()
seeds = P.replica_seeds(insts, R, "mfz-bn")
ctx = P.Context(0, "f32")
for it in range(3):
    t0 = time.perf_counter(); ctx.set_problems(insts); t1 = time.perf_counter()
    ctx.build_coupling(); t2 = time.perf_counter()
    res = ctx.solve(R, "mfz-bn", hp, seeds); t3 = time.perf_counter()
    tm = ctx.timing()
    print(f"set_problems {t1-t0:.3f}s build {t2-t1:.3f}s solve {t3-t2:.3f}s (device total {tm['total_ms']/1e3:.3f}s)")
