"""Dev tool: time-to-converge of every schedule x predictor on one workload (graph built once)."""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
from paper_1806_00762_b200 import pagestream as ps  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--algo", default="sssp")
    ap.add_argument("--scale", type=int, default=24)
    ap.add_argument("--pages", type=int, default=16)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--modes", default="baseline,reentry,double-buffer,pipelined,pipelined-fine")
    ap.add_argument("--preds", default="off,strong,weak")
    ap.add_argument("--uniform", action="store_true")
    a = ap.parse_args()
    args = bench.parse.__wrapped__() if hasattr(bench.parse, "__wrapped__") else None
    ns = argparse.Namespace(algo=a.algo, scale=a.scale, edge_factor=16, uniform=a.uniform,
                            pages=a.pages, seed=0, lean=True, graph="device")
    t0 = time.time()
    eng = ps.Engine(0)
    W = bench.workload(ns, eng)
    print(f"# build {time.time() - t0:.1f}s n={W['n']} m={W['m']}", flush=True)
    if not W["loaded"]:
        eng.load_csr(W["csr"], with_edges=False)
        eng.load_pages(W["pages"])
    kind = ps.AlgoKind(bench.ALGOS[a.algo])
    prog = ps.VertexProgram(kind, 0)
    for mode in a.modes.split(","):
        for pred in a.preds.split(","):
            cfg = ps.EngineConfig(predictor=ps.PredictorMode(bench.PREDS[pred]),
                                  clock=ps.ClockMode.WALL)
            cfg.schedule.kind = ps.ScheduleModeKind(bench.MODES[mode])
            eng.run(prog, cfg, want_values=False)
            ts = []
            for _ in range(a.reps):
                r = eng.run(prog, cfg, want_values=False)
                ts.append(r.metrics.device_seconds)
            m = r.metrics
            t = min(ts)
            print(json.dumps({"mode": mode, "pred": pred, "ms": round(t * 1e3, 3),
                              "gteps": round(W["m"] / t / 1e9, 2),
                              "passes": [m.dense_passes, m.sparse_passes, m.recovery_passes],
                              "edges_read": m.edges_read, "launches": m.kernel_launches}),
                  flush=True)
    ms, e = eng.bench_pull_sweep(kind, 20)
    per = 12 if kind == ps.AlgoKind.SSSP else 8
    print(json.dumps({"sweep_ms": round(ms, 4), "edges": e,
                      "GBps": round((per * e + 8 * W["n"]) / ms / 1e6, 1)}), flush=True)


if __name__ == "__main__":
    main()
