"""Dev tool: time the phases of the e2e call (load_csr, load_pages incl. tile build,
device CSR derivation, run, D2H) on the bench workload."""
import argparse
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import bench  # noqa: E402
from paper_1806_00762_b200 import _native as N  # noqa: E402
from paper_1806_00762_b200 import pagestream as ps  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--scale", type=int, default=24)
ap.add_argument("--algo", default="sssp")
ap.add_argument("--uniform", action="store_true")
a = ap.parse_args()
ns = argparse.Namespace(algo=a.algo, scale=a.scale, edge_factor=16, uniform=a.uniform, pages=16,
                        seed=0, lean=True, graph="device")
W = bench.workload(ns)
csr, pages = W["csr"], W["pages"]
eng = ps.Engine(0)
cfg = ps.EngineConfig(predictor=ps.PredictorMode.STRONG, clock=ps.ClockMode.WALL)
prog = (ps.make_sssp(0, W["n"], True) if a.algo == "sssp" else
        ps.make_cc() if a.algo == "cc" else ps.make_bfs(0, W["n"]))
vals = np.empty(W["n"], np.uint32)
for rep in range(3):
    t0 = time.time()
    eng.load_csr(csr, with_edges=False)
    t1 = time.time()
    eng.load_pages(pages)
    t2 = time.time()
    r = eng.run(prog, cfg, values_out=vals)
    t3 = time.time()
    print(f"load_csr {1e3*(t1-t0):.1f} ms  load_pages {1e3*(t2-t1):.1f} ms  "
          f"run+derive+d2h {1e3*(t3-t2):.1f} ms (device {1e3*r.metrics.device_seconds:.2f})", flush=True)
t0 = time.time()
eng.run(prog, cfg, values_out=vals)
print(f"run only (derived csr cached) {1e3*(time.time()-t0):.1f} ms", flush=True)
gb = N.C.c_double()
N.check(N.lib.sr_bench_h2d(0, 1 << 30, 3, N.C.byref(gb)))
print("h2d GB/s", gb.value)

for rep in range(4):
    t0 = time.time()
    r = eng.run_graph(csr, pages, prog, cfg, values_out=vals)
    print(f"run_graph {1e3*(time.time()-t0):.1f} ms (upload {1e3*r.metrics.upload_seconds:.1f} ms, "
          f"device {1e3*r.metrics.device_seconds:.2f} ms)", flush=True)
