"""Key metrics of every kernel in an ncu --set full report (csv raw page)."""
import csv
import subprocess
import sys

WANT = [
    ("gpu__time_duration.sum", "us", 1e-3),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "dram%", 1),
    ("dram__bytes_read.sum", "rdMB", 1e-6),
    ("dram__bytes_write.sum", "wrMB", 1e-6),
    ("lts__t_sector_hit_rate.pct", "L2hit%", 1),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "occ%", 1),
    ("launch__registers_per_thread", "regs", 1),
    ("launch__grid_size", "grid", 1),
    ("launch__occupancy_limit_registers", "limR", 1),
    ("smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio", "stall_lsb", 1),
    ("smsp__average_warps_issue_stalled_lg_throttle_per_issue_active.ratio", "stall_lgt", 1),
    ("smsp__average_warps_issue_stalled_drain_per_issue_active.ratio", "stall_drain", 1),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue%", 1),
]


def main(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h, units = rows[0], rows[1]
    idx = {n: h.index(n) for n, _, _ in WANT if n in h}
    kn = h.index("Kernel Name")
    print("kernel".ljust(48) + " ".join(lbl.rjust(9) for n, lbl, _ in WANT if n in idx))
    for r in rows[2:]:
        vals = []
        for n, lbl, sc in WANT:
            if n not in idx:
                continue
            v = r[idx[n]].replace(",", "")
            try:
                x = float(v)
                u = units[idx[n]]
                if n.startswith("dram__bytes"):
                    x *= {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
                elif n == "gpu__time_duration.sum":
                    x *= {"ns": 1, "nsecond": 1, "us": 1e3, "usecond": 1e3, "ms": 1e6, "msecond": 1e6}.get(u, 1)
                vals.append(f"{x * sc:9.2f}")
            except ValueError:
                vals.append(v[:9].rjust(9))
        print(r[kn].split("(")[0][:47].ljust(48) + " ".join(vals))


if __name__ == "__main__":
    main(sys.argv[1])
