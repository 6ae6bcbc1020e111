"""SASS evidence per hot kernel of libcimcs_gpu.so (cuobjdump, no GPU needed):
instruction-class counts that prove the Blackwell paths (UTC*MMA = tcgen05.mma,
LDTM = tcgen05.ld, UBLKCP = cp.async.bulk, DMMA = fp64 mma.sync, SYNCS = mbarrier)
plus registers / spills.
  python tools/sass_summary.py > profiles/r02_sass_summary.txt
Also counts BRA.U.ANY: zero means every tcgen05.mma / bulk copy is issued straight from
uniform registers (no per-instruction ELECT / R2UR / BRA.U.ANY loop).
"""
import collections
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2405_00366_b200", "libcimcs_gpu.so")
HOT = ["sym_step_kernel", "sym_update_kernel", "sym64_step_kernel", "sym64_update_kernel",
       "gram_tc_kernel", "gt_split_kernel", "cluster_loop_kernel", "mri_cluster_kernel",
       "gemv_fused_kernel", "gram128_kernel"]
CLASSES = ["UTCHMMA", "UTCQMMA", "UTCBAR", "LDTM", "STTM", "UBLKCP", "UTMALDG", "DMMA", "HMMA",
           "DFMA", "FFMA", "SYNCS", "LDS", "STS", "LDG", "STG", "SHFL", "BAR"]


def main():
    sass = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True).stdout
    res = subprocess.run(["cuobjdump", "--dump-resource-usage", LIB], capture_output=True,
                         text=True).stdout
    usage = {}
    cur = None
    for line in res.splitlines():
        m = re.search(r"Function (\S+):", line)
        if m:
            cur = m.group(1)
        elif cur and "REG:" in line:
            usage[cur] = " ".join(re.findall(r"(REG:\d+|STACK:\d+|SHARED:\d+|LOCAL:\d+)", line))
    funcs = re.split(r"\n\s+Function : ", sass)
    print("SASS instruction classes per hot kernel (cuobjdump -sass of "
          "paper_2405_00366_b200/libcimcs_gpu.so, sm_100a)")
    seen = collections.defaultdict(int)
    for f in funcs[1:]:
        name = f.split("\n", 1)[0].strip()
        hot = next((h for h in HOT if h in name), None)
        if hot is None or seen[hot] >= 2:  # two instantiations per kernel family suffice
            continue
        seen[hot] += 1
        ops = collections.Counter()
        for m in re.finditer(r"/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)", f):
            ops[m.group(1)] += 1
        cls = {c: sum(v for k, v in ops.items() if k.startswith(c)) for c in CLASSES}
        # waterfall loops around uniform-register instructions (an `if (lane == 0)` issue
        # path makes ptxas emit ELECT / R2UR.BROADCAST / BRA.U.ANY per UTCHMMA / UBLKCP)
        cls["BRA.U.ANY(waterfall loops)"] = len(re.findall(r"BRA\.U\.ANY", f))
        cls["ELECT"] = ops.get("ELECT", 0)
        cls["R2UR"] = ops.get("R2UR", 0)
        demangled = subprocess.run(["c++filt", name], capture_output=True, text=True).stdout.strip()
        print(f"\n{demangled}\n  {usage.get(name, '')}")
        print("  " + "  ".join(f"{c}={n}" for c, n in cls.items() if n))


if __name__ == "__main__":
    sys.exit(main())
