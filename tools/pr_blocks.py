"""Dev tool: PageRank RMAT-26 resident time vs source-block size (SERAPH_PR_BLOCK_VERTS)."""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_1806_00762_b200 import pagestream as ps  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--scale", type=int, default=26)
ap.add_argument("--blocks", default="0,4194304,8388608,16777216,33554432")
a = ap.parse_args()
W = bench.workload(argparse.Namespace(algo="pagerank", scale=a.scale, edge_factor=16,
                                      uniform=False, pages=16, seed=0, lean=True))
for blk in a.blocks.split(","):
    os.environ["SERAPH_PR_BLOCK_VERTS"] = blk
    with ps.Engine(0) as eng:
        eng.load_csr(W["csr"], with_edges=False)
        eng.load_pages(W["pages"])
        cfg = ps.EngineConfig(clock=ps.ClockMode.WALL, profile_kernels=True)
        eng.run(ps.make_pagerank(), cfg, want_values=False)
        ts = [eng.run(ps.make_pagerank(), cfg, want_values=False).metrics for _ in range(3)]
        t = min(m.device_seconds for m in ts)
        m = ts[-1]
        print(f"blk {blk:>9}: {t*1e3:8.2f} ms  {W['m']*20/t/1e9:7.1f} GTEPS  relax {m.relax_seconds*1e3:.1f} ms in {m.relax_launches} launches", flush=True)
