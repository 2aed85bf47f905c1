"""Dev/validation tool: the sharded world at full C4 scale on ONE GPU -- a
sr_group world of N ranks on cuda:0 (loopback exchange through host memory)
runs pagestream::run on the reference's uniform-27 instance and must end with
exactly the single-context labels (and the CC signature: one component,
label sum 0).  Exercises the sharded blocked sweeps (diagonal first, block-0
subgraph iteration, per-block probes), own-row CSR shards and the per-round
exchange at the size the SCALE runs use, without NCCL.

    python tools/group_scale_check.py [--world 2] [--peer] [--scale 27]
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
ap.add_argument("--world", type=int, default=2)
ap.add_argument("--peer", action="store_true")
ap.add_argument("--scale", type=int, default=27)
ap.add_argument("--algo", default="cc")
a = ap.parse_args()
n = 1 << a.scale
arena = N.PinnedArena()
t = time.time()
with ps.Engine(0) as scratch:
    scratch.generate_graph(a.scale, 16, *bench.UNIFORM, seed=0, symmetrize=a.algo == "cc",
                           weights=(1, 64, 1) if a.algo == "sssp" else None,
                           page_vertex_capacity=(n + 15) // 16, csr_edges=True)
    csr, pages = scratch.export_graph(arena, csr_edges=True)[:2]
print(f"# graph {time.time() - t:.1f} s, m={csr.num_edges()}", flush=True)
prog = {"cc": ps.make_cc(), "bfs": ps.make_bfs(0, n), "sssp": ps.make_sssp(0, n, True)}[a.algo]
cfg = ps.EngineConfig(predictor=ps.PredictorMode.STRONG, clock=ps.ClockMode.WALL)
with ps.Engine(0) as one:
    r1 = one.run_graph(csr, pages, prog, cfg)
print(f"# single context: {r1.metrics.device_seconds * 1e3:.2f} ms, {r1.metrics.passes} passes",
      flush=True)
with ps.Group([0] * a.world, exchange="peer" if a.peer else "allreduce") as g:
    t = time.time()
    rg = g.run_graph(csr, pages, prog, cfg)
    print(f"# group of {a.world}: call {time.time() - t:.1f} s, device "
          f"{rg.metrics.device_seconds * 1e3:.2f} ms, {rg.metrics.passes} passes", flush=True)
    infos = [g.graph_info(r) for r in range(a.world)]
same = np.array_equal(r1.values, rg.values)
sig = bench.value_signature(bench.ALGOS[a.algo], rg.values)
print({"bit_exact_vs_single": bool(same), "signature": sig,
       "ranks_hold_csr_rows": all(i["has_csr_edges"] for i in infos)})
sys.exit(0 if same else 1)
