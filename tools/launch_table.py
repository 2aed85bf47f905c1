"""Dev tool: per-launch table from an ncu --csv launch list (gpu__time_duration, dram bytes)."""
import csv
import sys
from collections import OrderedDict


def rows(path):
    with open(path) as fh:
        lines = [ln for ln in fh if ln.startswith('"')]
    return list(csv.DictReader(lines))


def main(path, full=False):
    per = OrderedDict()
    order = []
    for r in rows(path):
        key = (r["ID"], r["Kernel Name"])
        if key not in per:
            per[key] = {}
            order.append(key)
        v = r["Metric Value"].replace(",", "")
        try:
            per[key][r["Metric Name"]] = (float(v), r["Metric Unit"])
        except ValueError:
            pass
    tot = 0.0
    agg = OrderedDict()
    for key in order:
        m = per[key]
        t, u = m.get("gpu__time_duration.sum", (0.0, "ns"))
        t_us = t / 1000.0 if u == "ns" else (t * 1000.0 if u == "ms" else t)
        rd = m.get("dram__bytes_read.sum", (0.0, "byte"))
        wr = m.get("dram__bytes_write.sum", (0.0, "byte"))
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
        b = rd[0] * scale.get(rd[1], 1) + wr[0] * scale.get(wr[1], 1)
        tot += t_us
        name = key[1].split("(")[0]
        a = agg.setdefault(name, [0, 0.0, 0.0])
        a[0] += 1
        a[1] += t_us
        a[2] += b
        if full:
            print(f"{key[0]:>5} {t_us:10.1f} us {b / 1e9:8.3f} GB {b / max(t_us, 1e-9) / 1e3:8.1f} GB/s  {name}")
    print(f"total {tot:.1f} us")
    for name, (n, t, b) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{n:5d} {t:12.1f} us {t / tot * 100:5.1f}% {b / 1e9:9.3f} GB {b / max(t, 1e-9) / 1e3:8.1f} GB/s  {name}")


def to_json(path, out):
    import json
    import os
    agg = {}
    tot = 0.0
    for r in rows(path):
        if r["Metric Name"] != "gpu__time_duration.sum":
            continue
        v = float(r["Metric Value"].replace(",", ""))
        t_us = v / 1000.0 if r["Metric Unit"] == "ns" else (v * 1000.0 if r["Metric Unit"] == "ms" else v)
        name = r["Kernel Name"].split("(")[0].replace("seraph::<unnamed>::", "")
        a = agg.setdefault(name, [0, 0.0])
        a[0] += 1
        a[1] += t_us
        tot += t_us
    ks = [{"kernel": k, "launches": n, "total_us": round(t, 1), "share": round(t / tot, 4)}
          for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1])]
    with open(out, "w") as fh:
        json.dump({"source": os.path.basename(path), "total_us": round(tot, 1), "kernels": ks}, fh,
                  indent=1)


if __name__ == "__main__":
    if "--json" in sys.argv:
        to_json(sys.argv[1], sys.argv[sys.argv.index("--json") + 1])
    else:
        main(sys.argv[1], "--full" in sys.argv)
