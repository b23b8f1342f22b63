"""Summarise an ncu --csv launch list (gpu__time_duration.sum per launch) by kernel."""
import collections
import csv
import sys


def summarise(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    hdr, data = rows[hi], rows[hi + 1:]
    ki, vi, mi = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Name")
    ui = hdr.index("Metric Unit") if "Metric Unit" in hdr else None
    agg = collections.OrderedDict()
    for r in data:
        if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
            continue
        name = r[ki].split("(")[0].replace("void ", "")
        name = name.split("::")[-1]
        v = float(r[vi].replace(",", ""))
        if ui is not None and r[ui] == "usecond":
            v *= 1e3
        elif ui is not None and r[ui] == "msecond":
            v *= 1e6
        a = agg.setdefault(name, [0, 0.0])
        a[0] += 1
        a[1] += v
    tot = sum(v for _, v in agg.values())
    out = [f"{'kernel':40s} {'launches':>8s} {'avg_us':>9s} {'share':>7s}"]
    for k, (n, v) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        out.append(f"{k[:40]:40s} {n:8d} {v / n / 1e3:9.2f} {100 * v / tot:6.1f}%")
    return "\n".join(out)


if __name__ == "__main__":
    print(summarise(sys.argv[1]))
