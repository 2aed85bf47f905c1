"""Dev tool: one resident workload, one converge run, then K1 dense sweeps (ncu target)."""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
from paper_1806_00762_b200 import pagestream as ps  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--algo", default="sssp")
ap.add_argument("--scale", type=int, default=24)
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--converge", type=int, default=1)
ap.add_argument("--uniform", action="store_true")
a = ap.parse_args()
ns = argparse.Namespace(algo=a.algo, scale=a.scale, edge_factor=16, uniform=a.algo == "cc" and a.uniform,
                        pages=16, seed=0, graph="device", lean=False)
eng = ps.Engine(0)
W = bench.workload(ns, eng)
if not W["loaded"]:
    eng.load(W["csr"], W["pages"])
kind = ps.AlgoKind(bench.ALGOS[a.algo])
cfg = ps.EngineConfig(predictor=ps.PredictorMode.STRONG, clock=ps.ClockMode.WALL)
for _ in range(a.converge):
    r = eng.run(ps.VertexProgram(kind, 0), cfg, want_values=False)
ms, e = eng.bench_pull_sweep(kind, a.reps)
print("sweep ms", ms, "edges", e, "converge ms", r.metrics.device_seconds * 1e3)
