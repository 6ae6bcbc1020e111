"""Summarise an ncu launch list (`--metrics gpu__time_duration.sum --csv
--log-file X`) into per-kernel launches / total / share / average lines."""
import csv
import sys
from collections import OrderedDict


def main(path, header):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    h = rows[0]
    ik, im, iv = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
    agg = OrderedDict()
    for r in rows[1:]:
        if r[im] != "gpu__time_duration.sum":
            continue
        name = r[ik].split("(")[0].replace("void ", "")
        v = float(r[iv].replace(",", ""))
        unit = r[im + 1] if len(r) > im + 1 else ""
        if "Metric Unit" in h:
            unit = r[h.index("Metric Unit")]
        us = v / 1e3 if unit == "ns" else (v * 1e3 if unit == "ms" else v)
        n, t = agg.get(name, (0, 0.0))
        agg[name] = (n + 1, t + us)
    tot = sum(t for _, t in agg.values())
    print(header)
    for name, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"{name[:60]:60s} launches={n:6d} total_us={t:11.1f} share={100 * t / tot:5.1f}% "
              f"avg_us={t / n:9.1f}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else "")
