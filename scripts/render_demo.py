"""Renders the C3 pool caustic (T chain) on the receiver plane, specular and glossy (8 Beckmann offset samples,
alpha 0.05), with the deterministic splat renderer (spoly_render); writes PPM + PFM into profiles/ and prints the
render times.  Usage (GPU box): python scripts/render_demo.py [res]"""
import json
import os
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2405_13409_b200 import image_io, spoly  # noqa: E402
from paper_2405_13409_b200 import workloads as W  # noqa: E402

res = int(sys.argv[1]) if len(sys.argv) > 1 else 192
w = W.pool_c3(res=res)
ctx = spoly.Context(0)
ctx.upload_mesh(w.mesh)
ep = torch.as_tensor(w.endpoints, dtype=torch.float64, device="cuda")
it = torch.as_tensor(w.intensity, dtype=torch.float64, device="cuda")
out = {"workload": f"C3 pool, {res}x{res} receivers, {w.mesh.ntris} tris, chain T"}
for name, slopes in (("specular", None), ("glossy", W.beckmann_slopes(7, 8, w.mesh.ntris, 0.05))):
    ctx.render("T", ep, res, res, intensity=it, slopes=slopes, albedo=0.8, exposure=1.0)  # warm-up
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    rad, rgb = ctx.render("T", ep, res, res, intensity=it, slopes=slopes, albedo=0.8, exposure=1.0)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    m = float(rad.max())
    # the caustic's brightest pixel at code 255: re-tone-map with exposure 1 / max (same kernel)
    rad, rgb = ctx.render("T", ep, res, res, intensity=it, slopes=slopes, albedo=0.8, exposure=1.0 / m)
    image_io.write_ppm(os.path.join(ROOT, "profiles", f"render_pool_{name}.ppm"), rgb)
    image_io.write_pfm(os.path.join(ROOT, "profiles", f"render_pool_{name}.pfm"), rad)
    out[name] = {"samples": 1 if slopes is None else slopes.shape[0], "render_ms": dt * 1e3, "max_radiance": m,
                 "lit_pixels": int((rad > 0).sum())}
print(json.dumps(out))
