"""Dev tool: per-pass breakdown of one converge run (stats + per-kernel device time).

    python tools/pass_probe.py --algo sssp --scale 24
    ncu --profile-from-start off --metrics gpu__time_duration.sum --csv \
        python tools/pass_probe.py ...   # only the probed run is captured
"""
import argparse
import ctypes
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
from paper_1806_00762_b200 import pagestream as ps  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--algo", default="sssp")
    ap.add_argument("--scale", type=int, default=24)
    ap.add_argument("--pages", type=int, default=16)
    ap.add_argument("--uniform", action="store_true")
    ap.add_argument("--mode", default="baseline")
    ap.add_argument("--predictor", default="strong")
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--budget-gb", type=float, default=0.0)
    ap.add_argument("--window", type=int, default=8)
    ap.add_argument("--execution", default="density_switched",
                    choices=[e.name.lower() for e in ps.ExecutionPolicy])
    ap.add_argument("--sweep", default="", help="VAR=v1,v2,...: time one run per setting")
    ap.add_argument("--verify", action="store_true")
    a = ap.parse_args()
    n = 1 << a.scale
    quad = bench.UNIFORM if a.uniform else bench.RMAT
    gen = dict(seed=0, weights=(1, 64, 1) if a.algo == "sssp" else None,
               symmetrize=a.algo == "cc", page_vertex_capacity=(n + a.pages - 1) // a.pages)
    if a.budget_gb:  # out of core: build in a scratch context, load under the budget
        from paper_1806_00762_b200 import _native as N
        arena = N.PinnedArena()
        with ps.Engine(0) as scratch:
            scratch.generate_graph(a.scale, 16, *quad, csr_edges=True, **gen)
            host = scratch.export_graph(arena, csr_edges=a.algo != "pagerank")
        eng = ps.Engine(0, int(a.budget_gb * 2**30))
        eng.load_csr(host[0], with_edges=a.algo != "pagerank")
        eng.load_pages(host[1])
    else:
        eng = ps.Engine(0)
        eng.generate_graph(a.scale, 16, *quad, csr_edges=False, **gen)
    print(f"# n={n} m={eng.graph_info()['num_edges']}", flush=True)
    kind = ps.AlgoKind(bench.ALGOS[a.algo])
    prog = ps.VertexProgram(kind, 0)
    cfg = ps.EngineConfig(predictor=ps.PredictorMode(bench.PREDS[a.predictor]),
                          clock=ps.ClockMode.WALL, profile_kernels=True,
                          window_capacity=a.window,
                          execution=ps.ExecutionPolicy[a.execution.upper()])
    cfg.schedule.kind = ps.ScheduleModeKind(bench.MODES[a.mode])
    if a.sweep:
        var, vals = a.sweep.split("=", 1)
        base = None
        for v in vals.split(","):
            if v == "unset":
                os.environ.pop(var, None)
            else:
                os.environ[var] = v
            r = eng.run(prog, cfg, want_values=a.verify)  # builds per-setting structures
            extra = {}
            if a.verify and kind != ps.AlgoKind.PAGERANK:
                extra["violations"] = eng.verify_fixpoint(kind, r.values)
            if a.verify:
                got = r.ranks if kind == ps.AlgoKind.PAGERANK else r.values
                if base is None:
                    base = got.copy()
                elif kind == ps.AlgoKind.PAGERANK:
                    extra["max_diff_vs_first"] = float(abs(got.astype("f8") - base).max())
                else:
                    extra["equal_to_first"] = bool((got == base).all())
            ts = []
            for _ in range(a.reps):
                ts.append(eng.run(prog, cfg, want_values=False).metrics.device_seconds * 1e3)
            print(json.dumps({var: v, "ms": [round(t, 3) for t in ts], "first_ms":
                              round(r.metrics.device_seconds * 1e3, 3), **extra}), flush=True)
        return
    for _ in range(a.reps):
        r = eng.run(prog, cfg, want_values=False)
    cudart = ctypes.CDLL("libcudart.so")
    cudart.cudaProfilerStart()
    r = eng.run(prog, cfg, want_values=False)
    cudart.cudaDeviceSynchronize()
    cudart.cudaProfilerStop()
    m = r.metrics
    print(json.dumps({"ms": round(m.device_seconds * 1e3, 4),
                      "relax_ms": round(m.relax_seconds * 1e3, 4),
                      "relax_launches": m.relax_launches, "launches": m.kernel_launches,
                      "gathers": m.gathers, "edges_read": m.edges_read,
                      "bytes_transferred": m.bytes_transferred}))
    for st in m.per_pass:
        print(json.dumps({"pass": st.pass_index, "kind": int(st.kind), "attempts": st.attempts,
                          "valid": st.valid_updates, "skipped": st.skipped,
                          "edges": st.edges_read, "changed": st.changed_vertices}))


if __name__ == "__main__":
    main()
