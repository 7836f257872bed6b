"""One full-size C5 solve (1,048,576 receivers x 2,560-tri glass shell, TT) on one B200: demonstrates the
north_star sweep size runs through the chunked two-bounce cull; one timed solve after one warm-up solve
(a bench.py line at this size would take ~30 min with its 3 warm-up steps).  Prints one JSON line."""
import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2405_13409_b200 import spoly  # noqa: E402
from paper_2405_13409_b200 import workloads as W  # noqa: E402

res = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
w = W.shell_c5(res=res)
ctx = spoly.Context(0)
ctx.upload_mesh(w.mesh)
ep = torch.as_tensor(w.endpoints, dtype=torch.float64, device="cuda")
warm = w.subset(list(range(0, w.nqueries, 64)))  # warm-up on a 1/64 subsample (allocations, module load)
ctx.solve("TT", torch.as_tensor(warm.endpoints, dtype=torch.float64, device="cuda"))
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
t0 = time.perf_counter()
e0.record()
r = ctx.solve("TT", ep)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1)
rep = r.report
print(json.dumps({"config": f"C5 TT shell, {w.nqueries} receivers x {w.mesh.ntris} tris", "ms": ms,
                  "wall_s": time.perf_counter() - t0, "paths": r.n_solutions, "paths_per_s": r.n_solutions / (ms / 1e3),
                  "pairs_refined": rep["n_pairs_in"], "pairs_coarse": rep["n_pairs_coarse"],
                  "ms_cull": rep["ms_cull"], "ms_solve": rep["ms_solve"], "ms_reduce": rep["ms_reduce"],
                  "cull_tests": rep["n_cull_tests"], "flagged": rep["n_flagged"]}))
