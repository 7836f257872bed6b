import sys, os, json
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import numpy as np, torch
from paper_2405_13409_b200 import spoly, workloads as W
w = W.sphere_c4(res=128, level=4)
qs = [8256, 8300, 4000, 12000, 6000, 9000, 2100, 14100]
sub = w.subset(qs)
for lv in (3, 5):
    ctx = spoly.Context(0, spoly.default_config(cull_levels=lv))
    ctx.upload_mesh(sub.mesh)
    r = ctx.solve("TT", torch.as_tensor(sub.endpoints, device="cuda"))
    pq, pt = ctx.last_worklist()
    pq = pq.cpu().numpy().view(np.uint32); pt = pt.cpu().numpy().view(np.uint32)
    np.save(f"gpurun_out/c4wl_{lv}.npy", np.c_[pq, pt])
    print(lv, np.bincount(pq, minlength=len(qs)).tolist(), r.report["n_pairs_coarse"], flush=True)
    ctx.close()
