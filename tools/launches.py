"""Summarise an ncu launch list (csv): gpu__time_duration.sum per kernel, plus
DRAM bytes (dram__bytes_read.sum + dram__bytes_write.sum) and the achieved
DRAM GB/s when those metrics were collected."""
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
        a = agg.setdefault(n, {"ids": set(), "ns": 0.0, "bytes": 0.0})
        a["ids"].add(r["ID"])
        v = float(r["Metric Value"].replace(",", ""))
        if r["Metric Name"] == "gpu__time_duration.sum":
            a["ns"] += v * {"ns": 1, "nsecond": 1, "us": 1e3, "usecond": 1e3, "ms": 1e6, "msecond": 1e6}.get(
                r["Metric Unit"], 1)
        elif r["Metric Name"].startswith("dram__bytes"):
            a["bytes"] += v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(r["Metric Unit"], 1)
    tot = sum(v["ns"] for v in agg.values())
    out = [f"{'launches':>8} {'total us':>10} {'share':>6} {'us/launch':>9} {'DRAM MB/l':>9} {'GB/s':>7}  kernel"]
    for k, v in sorted(agg.items(), key=lambda x: -x[1]["ns"]):
        n = len(v["ids"])
        gbs = v["bytes"] / v["ns"] if v["ns"] else 0.0
        out.append(f"{n:8d} {v['ns'] / 1e3:10.1f} {100 * v['ns'] / tot:5.1f}% {v['ns'] / 1e3 / n:9.1f} "
                   f"{v['bytes'] / 1e6 / n:9.2f} {gbs:7.0f}  {k}")
    out.append(f"{sum(len(v['ids']) for v in agg.values()):8d} {tot / 1e3:10.1f}        total (excl. table init / torch)")
    return "\n".join(out)


if __name__ == "__main__":
    print(summary(sys.argv[1]))
