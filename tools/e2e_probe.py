"""Dev tool: time the phases of the e2e call (load_csr, load_pages incl. tiles and
the source-block prebuild, run incl. per-run preparation, D2H) on a bench graph.

    python tools/e2e_probe.py --algo pagerank --scale 26
"""
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
ap.add_argument("--pages", type=int, default=16)
a = ap.parse_args()
n = 1 << a.scale
arena = N.PinnedArena()
with ps.Engine(0) as scratch:
    scratch.generate_graph(a.scale, 16, *(bench.UNIFORM if a.uniform else bench.RMAT), seed=0,
                           weights=(1, 64, 1) if a.algo == "sssp" else None,
                           symmetrize=a.algo == "cc", page_vertex_capacity=(n + a.pages - 1) // a.pages,
                           csr_edges=False)
    csr, pages = scratch.export_graph(arena, csr_edges=False)[:2]
prog = {"sssp": ps.make_sssp(0, n, True), "cc": ps.make_cc(), "bfs": ps.make_bfs(0, n),
        "pagerank": ps.make_pagerank()}[a.algo]
cfg = ps.EngineConfig(predictor=ps.PredictorMode.STRONG, clock=ps.ClockMode.WALL)
eng = ps.Engine(0)
for rep in range(3):
    t = time.time()
    r = eng.run_graph(csr, pages, prog, cfg)
    print(f"run_graph {1e3*(time.time()-t):.1f} ms (upload {1e3*r.metrics.upload_seconds:.1f} ms, "
          f"device {1e3*r.metrics.device_seconds:.2f} ms, wall {1e3*r.metrics.wall_seconds:.1f} ms)",
          flush=True)
t = time.time()
r = eng.run(prog, cfg)
print(f"run only {1e3*(time.time()-t):.1f} ms (device {1e3*r.metrics.device_seconds:.2f} ms)")

# pageable copies (what the C++ drop-in passes): the same call and its phases
csr_p = ps.CsrGraph(n, np.array(csr.out_offsets), csr.out_neighbors, csr.out_weights)
pages_p = ps.PageSet(pages.num_vertices, pages.page_vertex_capacity, pages.weighted,
                     [ps.CscPage(p.vertex_begin, p.vertex_end, np.array(p.in_offsets),
                                 np.array(p.in_sources), np.array(p.in_weights))
                      for p in pages.pages])
out = np.zeros(n, np.float32 if a.algo == "pagerank" else np.uint32)
for rep in range(3):
    t = time.time()
    r = eng.run_graph(csr_p, pages_p, prog, cfg, values_out=out)
    print(f"pageable run_graph {1e3*(time.time()-t):.1f} ms (upload {1e3*r.metrics.upload_seconds:.1f}"
          f" ms, device {1e3*r.metrics.device_seconds:.2f} ms)", flush=True)
for rep in range(2):
    t0 = time.time()
    eng.load_csr(csr_p, with_edges=False)
    t1 = time.time()
    eng.load_pages(pages_p)
    t2 = time.time()
    r = eng.run(prog, cfg, values_out=out)
    t3 = time.time()
    print(f"pageable phases: load_csr {1e3*(t1-t0):.1f} load_pages {1e3*(t2-t1):.1f} "
          f"run+d2h {1e3*(t3-t2):.1f} ms", flush=True)
