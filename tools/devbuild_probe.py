"""Dev tool: time the device-side generate+build (sr_generate_graph) and the export."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_1806_00762_b200 import pagestream as ps  # noqa: E402

for scale, quad, weights, sym in [(24, (0.57, 0.19, 0.19, 0.05), (1, 64, 1), False),
                                  (26, (0.57, 0.19, 0.19, 0.05), None, False),
                                  (27, (0.25,) * 4, None, True)]:
    with ps.Engine(0) as eng:
        for csr_edges in (False, True):
            t = time.time()
            eng.generate_graph(scale, 16, *quad, seed=0, weights=weights, symmetrize=sym,
                               csr_edges=csr_edges)
            tb = time.time() - t
            t = time.time()
            if csr_edges and scale < 27:
                eng.export_graph()
            te = time.time() - t
            print(f"scale {scale} sym {sym} csr_edges {csr_edges}: build {tb:.2f}s export {te:.2f}s "
                  f"{eng.graph_info()}", flush=True)
