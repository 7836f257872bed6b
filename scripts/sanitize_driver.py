"""Small invocations of every kernel family for compute-sanitizer (memcheck / racecheck / synccheck / initcheck):
one bounce R and T with and without the cull (phase 1, deep jobs, both path kernels), two bounces RR/TT/RT/TR via
tuple lists and via the pair cull (build, bin, scan incl. n > 32, path), visibility, both deterministic orders."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import torch  # noqa: E402

from paper_2405_13409_b200 import spoly, workloads as W  # noqa: E402
from planted import planted_many  # noqa: E402


def run(mesh, chain, ep, cfg=None, off=None, ids=None, occ=None):
    ctx = spoly.Context(0, cfg)
    ctx.upload_mesh(mesh)
    if occ is not None:
        ctx.upload_occluders(occ)
    e = torch.as_tensor(np.ascontiguousarray(ep), dtype=torch.float64, device="cuda")
    o = None if off is None else torch.as_tensor(off.astype(np.int32), device="cuda")
    t = None if ids is None else torch.as_tensor(ids.astype(np.int32), device="cuda")
    r = ctx.solve(chain, e, None, o, t)
    torch.cuda.synchronize()
    n = r.n_solutions
    ctx.close()
    print(chain, n, flush=True)


w = W.glints_c2(res=16)
run(w.mesh, "R", w.endpoints)
os.environ["SPOLY_SORT_ORDER"] = "0"
run(w.mesh, "R", w.endpoints)
os.environ.pop("SPOLY_SORT_ORDER")
w = W.pool_c3(res=16, nverts_side=65)
run(w.mesh, "T", w.endpoints)
w = W.patch_c1()
run(w.mesh, "R", w.endpoints, cfg=spoly.default_config(cull=0))
for chain in ("RR", "TT", "RT", "TR"):
    cases = planted_many(5, chain, 6, size=0.15)
    pos = np.concatenate([c[0].pos for c in cases])
    nrm = np.concatenate([c[0].nrm for c in cases])
    tri = np.concatenate([c[0].tri + 6 * i for i, c in enumerate(cases)]).astype(np.uint32)
    mesh = W.Mesh(pos, nrm, tri, cases[0][0].eta_front, cases[0][0].eta_back)
    ep = np.array([[c[2], c[3]] for c in cases])
    off = np.arange(len(cases) + 1, dtype=np.uint32)
    ids = np.arange(2 * len(cases), dtype=np.uint32)
    run(mesh, chain, ep, off=off, ids=ids)
w = W.sphere_c4(res=4, level=1)  # n > 32 tuples: the shared-memory scan
run(w.mesh, "TT", w.endpoints)
w = W.mirrors_rr(res=4, quads=8)
run(w.mesh, "RR", w.endpoints, cfg=spoly.default_config(visibility=1))
print("sanitize driver done", flush=True)
