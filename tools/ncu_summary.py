"""Summarise an ncu report (read here, no GPU) into profiles/<name>.json/.txt."""
import csv
import io
import json
import subprocess
import sys


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    h, units = r[0], r[1]
    rows = [dict(zip(h, row)) for row in r[2:]]
    return rows, dict(zip(h, units))


def num(x):
    try:
        return float(str(x).replace(",", ""))
    except Exception:
        return None


KEYS = [
    "Kernel Name", "gpu__time_duration.sum", "sm__cycles_active.avg", "dram__bytes_read.sum",
    "dram__bytes_write.sum", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
    "lts__t_bytes.sum", "smsp__cycles_active.avg", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
]


STEP = ("sym_step_kernel", "sym_update_kernel", "mri_cluster_kernel")


def main(rep, name, note=""):
    rows, units = raw(rep)
    out = []
    for d in rows:
        e = {k: d.get(k) for k in KEYS if k in d}
        stalls = {k.replace("smsp__pcsamp_warps_issue_stalled_", ""): num(v) for k, v in d.items()
                  if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued")}
        tot = sum(v for v in stalls.values() if v) or 1.0
        e["stall_pct"] = {k: round(100 * v / tot, 1) for k, v in sorted(stalls.items(), key=lambda x: -(x[1] or 0))[:8] if v}
        rb, wb = num(d.get("dram__bytes_read.sum")), num(d.get("dram__bytes_write.sum"))
        ur, uw = units.get("dram__bytes_read.sum", ""), units.get("dram__bytes_write.sum", "")
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
        if rb is not None and wb is not None:
            e["dram_bytes_per_launch"] = rb * scale.get(ur, 1) + wb * scale.get(uw, 1)
        e["units"] = {k: units.get(k) for k in KEYS if k in units}
        out.append(e)
    summary = {"report": rep, "note": note, "kernels": out}
    if out:  # one step = the step kernels captured (setup kernels such as the gram
        # scale / w conversion launched once per call are listed but not counted)
        step = [k for k in out if any(s in (k.get("Kernel Name") or "") for s in STEP)] or out
        vals = [k.get("dram_bytes_per_launch") for k in step]
        summary["step_kernels"] = [k.get("Kernel Name") for k in step]
        summary["dram_bytes_per_launch"] = sum(v for v in vals if v) if all(vals) else vals[0]
    with open(f"profiles/{name}.json", "w") as f:
        json.dump(summary, f, indent=1)
    print(json.dumps(summary, indent=1)[:3000])


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], sys.argv[3] if len(sys.argv) > 3 else "")
