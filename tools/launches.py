"""Summarise an ncu --metrics gpu__time_duration.sum launch list (csv)."""
import collections
import csv
import sys


def summary(path, skip_names=("init_table", "elementwise")):
    lines = open(path).read().splitlines()
    i = [k for k, l in enumerate(lines) if l.startswith('"ID"')][0]
    rows = list(csv.DictReader(lines[i:]))
    agg = collections.OrderedDict()
    for r in rows:
        n = r["Kernel Name"].split("(")[0][:90]
        if any(s in n for s in skip_names):
            continue
        a = agg.setdefault(n, [0, 0.0])
        a[0] += 1
        a[1] += float(r["Metric Value"]) / 1e3
    tot = sum(v[1] for v in agg.values())
    out = [f"{'launches':>8} {'total us':>10} {'share':>6}  kernel"]
    for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
        out.append(f"{v[0]:8d} {v[1]:10.1f} {100 * v[1] / tot:5.1f}%  {k}")
    out.append(f"{sum(v[0] for v in agg.values()):8d} {tot:10.1f}        total (excl. table init / torch)")
    return "\n".join(out)


if __name__ == "__main__":
    print(summary(sys.argv[1]))
