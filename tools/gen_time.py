"""Host generation time of config 4's instance (the reference stream, bit-exact)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2405_00366_b200 as P
N = int(sys.argv[1]) if len(sys.argv) > 1 else 100_000
t = time.perf_counter()
insts = P.gen_instances(N, [(0.5, 0.05, 0.01, 7)])
print(f"host gen_instance N={N}: {time.perf_counter() - t:.1f} s on {os.cpu_count()} cores")
