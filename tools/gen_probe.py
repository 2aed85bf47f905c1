"""Stage timings of the device graph generator/build (SERAPH_TIMING=1)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1806_00762_b200 import pagestream as ps  # noqa: E402

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 27
uniform = len(sys.argv) > 2 and sys.argv[2] == "u"
os.environ["SERAPH_TIMING"] = "1"
q = (0.25,) * 4 if uniform else (0.57, 0.19, 0.19, 0.05)
with ps.Engine(0) as eng:
    for rep in range(2):
        t = time.time()
        eng.generate_graph(scale, 16, *q, seed=0, symmetrize=uniform,
                           weights=None if uniform else (1, 64, 1),
                           page_vertex_capacity=(1 << scale) // 16, csr_edges=False)
        print(f"rep {rep}: generate_graph total {time.time() - t:.3f} s", flush=True)
