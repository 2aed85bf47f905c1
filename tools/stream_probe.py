"""Dev tool: how busy the host link is during an out-of-core run (wall trace of
the copy stream: union of XFER_START..XFER_END intervals / run time)."""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
from paper_1806_00762_b200 import _native as N  # noqa: E402
from paper_1806_00762_b200 import pagestream as ps  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--algo", default="pagerank")
ap.add_argument("--scale", type=int, default=26)
ap.add_argument("--pages", type=int, default=256)
ap.add_argument("--window", type=int, default=4)
ap.add_argument("--budget-gb", type=float, default=2.0)
ap.add_argument("--mode", default="reentry")
ap.add_argument("--pr-iters", type=int, default=20)
a = ap.parse_args()
ns = argparse.Namespace(algo=a.algo, scale=a.scale, edge_factor=16, uniform=False, pages=a.pages,
                        seed=0, lean=False, graph="device")
W = bench.workload(ns)
eng = ps.Engine(0, int(a.budget_gb * 2**30))
eng.load_csr(W["csr"], with_edges=True)
eng.load_pages(W["pages"])
prog = ps.VertexProgram(ps.AlgoKind(bench.ALGOS[a.algo]), 0)
cfg = ps.EngineConfig(clock=ps.ClockMode.WALL, window_capacity=a.window,
                      pr_iterations=a.pr_iters, predictor=ps.PredictorMode.STRONG)
cfg.schedule.kind = ps.ScheduleModeKind(bench.MODES[a.mode])
eng.run(prog, cfg, want_values=False)
cfg.record_trace = True
r = eng.run(prog, cfg, want_values=False)
ev = r.trace
starts = {}
iv = []
kern = []
for e in ev:
    k = int(e.kind)
    if k == 0:
        starts.setdefault(e.page_id, []).append(e.time)
    elif k == 1 and starts.get(e.page_id):
        iv.append((starts[e.page_id].pop(0), e.time))
    elif k in (2, 4):
        starts.setdefault(("k", e.page_id), []).append(e.time)
    elif k == 3 and starts.get(("k", e.page_id)):
        kern.append((starts[("k", e.page_id)].pop(0), e.time))


def union(x):
    x = sorted(x)
    tot, cur_s, cur_e = 0.0, None, None
    for s, e in x:
        if cur_e is None or s > cur_e:
            if cur_e is not None:
                tot += cur_e - cur_s
            cur_s, cur_e = s, e
        else:
            cur_e = max(cur_e, e)
    if cur_e is not None:
        tot += cur_e - cur_s
    return tot


t0 = min(e.time for e in ev)
t1 = max(e.time for e in ev)
gb = N.C.c_double()
N.check(N.lib.sr_bench_h2d(0, 1 << 30, 3, N.C.byref(gb)))
gb18 = N.C.c_double()
N.check(N.lib.sr_bench_h2d(0, 18 << 20, 5, N.C.byref(gb18)))
print(json.dumps({"run_s": r.metrics.device_seconds, "trace_span_s": t1 - t0,
                  "xfers": len(iv), "link_busy_s": union(iv), "kernel_busy_s": union(kern),
                  "bytes": r.metrics.bytes_transferred,
                  "gbps_while_busy": r.metrics.bytes_transferred / max(union(iv), 1e-9) / 1e9,
                  "h2d_1GiB_gbps": gb.value, "h2d_18MiB_gbps": gb18.value}))
