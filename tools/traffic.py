"""From an ncu launch list with gpu__time_duration.sum, dram__bytes_read.sum
and dram__bytes_write.sum per launch (tools/gpu_prof3.sh), write
  profiles/traffic.json  — DRAM bytes per phase span (bench.py's roofline `traffic`)
  a per-kernel summary (stdout): launches, time share, DRAM bytes per launch.
Phase -> kernels (one rank): merge = k_copy_rows<MergeMap> (one span per launch);
co_update = the whole update of one iteration (k_grad_ptrs, SgdPlanOp scan,
k_sgd_single, k_sgd_flat, k_sgd_combine, or the stream kernel k_sgd_stream;
one span per iteration)."""
import collections
import csv
import json
import sys

UPDATE = ("k_grad_ptrs", "k_sgd_single", "k_sgd_flat", "k_sgd_warp", "k_sgd_combine", "k_sgd_stream")  # the plan scan runs on L (one rank)


def load(path):
    lines = open(path).read().splitlines()
    i = [k for k, l in enumerate(lines) if l.startswith('"ID"')][0]
    per = collections.OrderedDict()
    for r in csv.DictReader(lines[i:]):
        d = per.setdefault(r["ID"], {"name": r["Kernel Name"].split("(")[0]})
        v = float(r["Metric Value"].replace(",", ""))
        unit = r["Metric Unit"]
        if r["Metric Name"].startswith("dram__bytes"):
            v *= {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
        elif unit == "usecond":
            v *= 1e3
        elif unit == "msecond":
            v *= 1e6
        d[r["Metric Name"]] = v
    return list(per.values())


def main(path, out_json="profiles/traffic.json", key="n1"):
    ks = [k for k in load(path) if "init_table" not in k["name"] and "at::" not in k["name"]]
    agg = collections.OrderedDict()
    for k in ks:
        a = agg.setdefault(k["name"], [0, 0.0, 0.0])
        a[0] += 1
        a[1] += k.get("gpu__time_duration.sum", 0.0) / 1e3
        a[2] += k.get("dram__bytes_read.sum", 0.0) + k.get("dram__bytes_write.sum", 0.0)
    tot = sum(v[1] for v in agg.values())
    print(f"{'launches':>8} {'total us':>10} {'share':>6} {'DRAM MB/launch':>15}  kernel")
    for n, v in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{v[0]:8d} {v[1]:10.1f} {100 * v[1] / tot:5.1f}% {v[2] / v[0] / 1e6:15.2f}  {n[:90]}")
    merge = [k for k in ks if "MergeMap" in k["name"]]
    upd = [k for k in ks if any(u in k["name"] for u in UPDATE)]
    # one update per iteration: the stream kernel's launches (else the older
    # single + warp pair, one k_sgd_single per iteration)
    iters = sum(1 for k in ks if "k_sgd_stream" in k["name"]) or sum(1 for k in ks if "k_sgd_single" in k["name"])
    dram = lambda L: sum(k.get("dram__bytes_read.sum", 0) + k.get("dram__bytes_write.sum", 0) for k in L)  # noqa: E731
    res = {}
    if merge:
        res["merge"] = int(dram(merge) / len(merge))
    if iters:
        res["co_update"] = int(dram(upd) / iters)
    try:
        data = json.load(open(out_json))
    except (OSError, ValueError):
        data = {}
    data[key] = res
    data["source"] = data.get("source", {})
    data["source"][key] = (f"{path}: ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,"
                           "dram__bytes_write.sum (cold cache, serialised launches)")
    json.dump(data, open(out_json, "w"), indent=1)
    print(json.dumps(res))


if __name__ == "__main__":
    main(*sys.argv[1:])
