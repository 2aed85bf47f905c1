"""Summarise ncu evidence into profiles/ (tracked):

  python tools/ncu_summary.py report <file.ncu-rep> <key> <tag>
      -> profiles/<tag>_k1.json and updates profiles/ncu_summary.json[key]
         (dram bytes per launch read by bench.py as roofline.traffic)
  python tools/ncu_summary.py launches <launches.csv> <tag>
      -> profiles/<tag>_launches.json: per-kernel count, total time, share
"""
import csv
import json
import os
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tools"))
PROF = os.path.join(ROOT, "profiles")


def to_bytes(val, unit):
    mult = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
    return float(val.replace(",", "")) * mult.get(unit, 1)


def report(path, key, tag):
    import ncu_report
    ds = ncu_report.read(path)
    d = ds[0]
    ms = [float(x["gpu__time_duration.sum"][0]) *
          {"ns": 1e-6, "us": 1e-3, "ms": 1.0}.get(x["gpu__time_duration.sum"][1], 1.0) for x in ds]
    rds = [to_bytes(*x["dram__bytes_read.sum"]) for x in ds]
    wrs = [to_bytes(*x["dram__bytes_write.sum"]) for x in ds]
    rd, wr = sum(rds) / len(ds), sum(wrs) / len(ds)
    out = {"source": os.path.basename(path), "kernel": d["kernel"], "launches": len(ds),
           "duration_ms": sum(ms) / len(ds), "per_launch_ms": ms,
           "dram_bytes_read": rd, "dram_bytes_write": wr, "dram_bytes_per_launch": rd + wr,
           "metrics_per_launch": [{k: v for k, v in x.items() if k != "kernel"} for x in ds]}
    os.makedirs(PROF, exist_ok=True)
    with open(os.path.join(PROF, f"{tag}_k1.json"), "w") as fh:
        json.dump(out, fh, indent=1)
    summ_path = os.path.join(PROF, "ncu_summary.json")
    summ = json.load(open(summ_path)) if os.path.exists(summ_path) else {}
    summ[key] = {"tag": tag, "kernel": d["kernel"], "duration_ms": out["duration_ms"],
                 "dram_bytes_per_launch": rd + wr,
                 "note": f"mean over the {len(ds)} captured launches of one converge run ({out['source']})"}
    with open(summ_path, "w") as fh:
        json.dump(summ, fh, indent=1)
    print(json.dumps(summ[key]))


def launches(path, tag):
    rows = list(csv.reader(open(path)))
    hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hdr]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    mi = h.index("Metric Name") if "Metric Name" in h else None
    seq = []  # (kernel, ns) in launch order, duration rows only
    for r in rows[hdr + 1:]:
        if len(r) <= vi or (mi is not None and r[mi] != "gpu__time_duration.sum"):
            continue
        try:
            v = float(r[vi].replace(",", ""))
        except ValueError:
            continue
        seq.append((r[ki].split("(")[0].replace("void ", "").replace("unnamed>::", ""), v))

    def table(part):
        agg = defaultdict(lambda: [0, 0.0])
        for name, v in part:
            agg[name][0] += 1
            agg[name][1] += v
        tot = sum(v[1] for v in agg.values()) or 1.0
        return {"total_us": round(tot / 1e3, 1),
                "kernels": [{"kernel": k, "launches": c, "total_us": round(t / 1e3, 1),
                             "share": round(t / tot, 4)}
                            for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1])]}

    # one converge run: from the last init_values_kernel up to the next
    # non-run kernel (fixpoint verification, graph export ...)
    starts = [i for i, (k, _) in enumerate(seq) if "init_values_kernel" in k]
    run = []
    if starts:
        for k, v in seq[starts[-1]:]:
            if any(x in k for x in ("verify_kernel", "bench_pull", "flush")):
                break
            run.append((k, v))
    out = {"source": os.path.basename(path), "whole_process": table(seq),
           "last_converge_run": table(run)}
    out.update(out["whole_process"])
    with open(os.path.join(PROF, f"{tag}_launches.json"), "w") as fh:
        json.dump(out, fh, indent=1)
    print("last converge run: %.1f us" % out["last_converge_run"]["total_us"])
    for k in out["last_converge_run"]["kernels"]:
        print(f"{k['kernel']:45s} {k['launches']:5d} {k['total_us']:10.1f}us {100 * k['share']:5.1f}%")


if __name__ == "__main__":
    if sys.argv[1] == "report":
        report(sys.argv[2], sys.argv[3], sys.argv[4])
    else:
        launches(sys.argv[2], sys.argv[3])
