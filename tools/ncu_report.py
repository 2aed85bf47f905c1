"""Dev tool: key metrics of an ncu --set full report (one kernel launch)."""
import csv
import json
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
        "l1tex__t_sector_hit_rate.pct", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__throughput.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "launch__grid_size",
        "sm__cycles_elapsed.avg.per_second"]


def read(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h, u = rows[0], rows[1]
    res = []
    for v in rows[2:]:
        d = {"kernel": v[h.index("Kernel Name")]}
        for k in KEYS:
            if k in h:
                d[k] = (v[h.index(k)], u[h.index(k)])
        stalls = {}
        for i, w in enumerate(h):
            if w.startswith("smsp__average_warps_issue_stalled_") and w.endswith("_per_issue_active.ratio"):
                try:
                    if float(v[i]) > 0.1:
                        stalls[w[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]] = float(v[i])
                except ValueError:
                    pass
        d["stalls_per_issue"] = stalls
        res.append(d)
    return res


if __name__ == "__main__":
    for d in read(sys.argv[1]):
        print(json.dumps(d, indent=1))
