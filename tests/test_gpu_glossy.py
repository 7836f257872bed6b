"""GPU (C-ABI) vs oracle parity of the glossy extension (spoly_set_normal_offsets, reading R28)
and of the deterministic splat renderer (spoly_render).  Needs a B200."""
import numpy as np
import pytest

import parity
from paper_2405_13409_b200 import workloads as W
from test_glossy_render import image_source_mask

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch_cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch


@pytest.fixture(scope="module")
def sp(torch_cuda):
    from paper_2405_13409_b200 import spoly
    spoly.lib()
    return spoly


def _solve(ctx, torch, chain, ep):
    e = torch.as_tensor(np.ascontiguousarray(ep), dtype=torch.float64, device="cuda")
    r = ctx.solve(chain, e)
    out = r.to_numpy()
    out["report"] = r.report
    wl = ctx.last_worklist()
    out["worklist"] = (wl[0].cpu().numpy().view(np.uint32),
                       wl[1].cpu().numpy().view(np.uint32).reshape(-1, len(chain)))
    return out


@pytest.mark.parametrize("name,alpha,tol", [("C2", 0.1, 1e-5), ("C3", 0.05, 1e-5), ("C5RR", 0.03, 1e-4),
                                            ("C4", 0.02, 1e-4)])
def test_glossy_solve_parity(sp, torch_cuda, orc, name, alpha, tol):
    # one offset sample on a one-bounce glint / caustic subset and on the two-bounce mirrors: the GPU solve after
    # spoly_set_normal_offsets equals the oracle's solve of the perturbed (de-indexed) surface
    w = {"C2": lambda: W.glints_c2(res=24), "C3": lambda: W.pool_c3(res=32),
         "C5RR": lambda: W.mirrors_rr(res=16, quads=16).subset(np.arange(0, 256, 2)),
         "C4": lambda: W.sphere_c4(res=32).subset(np.arange(0, 1024, 32))}[name]()
    sl = W.beckmann_slopes(11, 1, w.mesh.ntris, alpha)[0]
    ctx = sp.Context(0)
    ctx.upload_mesh(w.mesh)
    ctx.set_normal_offsets(sl)
    g = _solve(ctx, torch_cuda, w.chain, w.endpoints)
    m = orc.perturb_normals(w.mesh, sl)
    o = orc.solve(m, w.chain, w.endpoints)
    st = parity.compare(o, g, w.nqueries, tol_bary=tol, min_compared=10, label=f"glossy {name}")
    assert st["compared_solutions"] >= 10
    # restoring the uploaded normals restores the specular result bit for bit
    ctx.set_normal_offsets(None)
    a = _solve(ctx, torch_cuda, w.chain, w.endpoints)
    ctx.close()
    ctx2 = sp.Context(0)
    ctx2.upload_mesh(w.mesh)
    b = _solve(ctx2, torch_cuda, w.chain, w.endpoints)
    ctx2.close()
    for k in ("query", "tuple", "bary", "per_query"):
        assert np.array_equal(a[k], b[k]), k


def test_normal_offsets_bad_args(sp, torch_cuda):
    w = W.patch_c1()
    ctx = sp.Context(0)
    with pytest.raises(sp.SpolyError):
        ctx.set_normal_offsets(np.zeros((w.mesh.ntris, 2)))  # no mesh yet
    ctx.upload_mesh(w.mesh)
    with pytest.raises(sp.SpolyError):
        ctx.set_normal_offsets(np.zeros((w.mesh.ntris + 1, 2)))
    bad = np.zeros((w.mesh.ntris, 2))
    bad[3, 1] = np.nan
    with pytest.raises(sp.SpolyError):
        ctx.set_normal_offsets(bad)
    ctx.close()


def test_render_mirror_caustic(sp, torch_cuda, orc):
    # SPEC S:668 image-source mask (IoU = 1) and closed-form radiance on the GPU, and parity with the oracle render
    res = 96
    w, lit, L, margin = image_source_mask(res)
    ctx = sp.Context(0)
    ctx.upload_mesh(w.mesh)
    e = torch_cuda.as_tensor(w.endpoints, dtype=torch_cuda.float64, device="cuda")
    it = torch_cuda.as_tensor(w.intensity, dtype=torch_cuda.float64, device="cuda")
    rad, rgb = ctx.render("R", e, res, res, intensity=it, albedo=0.8, exposure=2.0)
    rad = rad.cpu().numpy().ravel()
    rgb = rgb.cpu().numpy().reshape(-1, 3)
    ctx.close()
    clear = margin > 1e-6
    got = rad > 0
    assert lit.sum() > 100 and np.sum(got & lit & clear) == np.sum((got | lit) & clear)
    assert np.allclose(rad[lit & clear], 0.8 / np.pi / L[lit & clear] ** 2, rtol=1e-8)
    orad, orgb, _ = orc.render(w.mesh, "R", w.endpoints, res, res, intensity=w.intensity, albedo=0.8, exposure=2.0)
    assert np.allclose(rad, orad.ravel(), rtol=1e-10, atol=0)
    _codes_agree(rgb, orgb.reshape(-1, 3), orad.ravel(), 2.0)


def _codes_agree(rgb, orgb, orad, exposure):
    # the code is an integer decided by FP64 arithmetic on values that agree to ~1e-12: equal except exactly at a
    # rounding boundary (255 v^(1/2.2) within 1e-6 of k + 1/2)
    x = 255.0 * np.minimum(1, np.maximum(0, exposure * orad)) ** (1 / 2.2)
    edge = np.abs(x - np.floor(x) - 0.5) < 1e-6
    assert np.all(rgb[:, 0] == rgb[:, 1]) and np.all(rgb[:, 0] == rgb[:, 2])
    diff = rgb[:, 0] != orgb[:, 0]
    assert not np.any(diff & ~edge), np.flatnonzero(diff & ~edge)[:10]


@pytest.mark.parametrize("name,chain,S,alpha", [("C2", "R", 3, 0.08), ("C3", "T", 2, 0.05)])
def test_render_glossy_parity(sp, torch_cuda, orc, name, chain, S, alpha):
    # S offset samples (Beckmann slopes, reading R28): the GPU render equals the oracle render on every pixel whose
    # tuples carry no flag in any sample
    res = 24
    w = {"C2": lambda: W.glints_c2(res=res), "C3": lambda: W.pool_c3(res=res)}[name]()
    sl = W.beckmann_slopes(21, S, w.mesh.ntris, alpha)
    ctx = sp.Context(0)
    ctx.upload_mesh(w.mesh)
    e = torch_cuda.as_tensor(w.endpoints, dtype=torch_cuda.float64, device="cuda")
    it = torch_cuda.as_tensor(w.intensity, dtype=torch_cuda.float64, device="cuda")
    rad, rgb = ctx.render(chain, e, res, res, intensity=it, slopes=sl, albedo=0.7, exposure=1.0)
    rad = rad.cpu().numpy().ravel()
    rgb = rgb.cpu().numpy().reshape(-1, 3)
    # the render restored the uploaded normals
    after = ctx.solve(chain, e, it).to_numpy()
    ctx.close()
    orad, orgb, rs = orc.render(w.mesh, chain, w.endpoints, res, res, intensity=w.intensity, slopes=sl, albedo=0.7)
    spec = orc.solve(w.mesh, chain, w.endpoints, w.intensity)
    fq = {int(q) for q in spec.flagged_query} | set(int(q) for q in after["flagged_query"])
    assert np.allclose(after["per_query"][[q for q in range(w.nqueries) if q not in fq]],
                       spec.per_query[[q for q in range(w.nqueries) if q not in fq]], rtol=1e-4, atol=0)
    flagged = set()
    for r in rs:
        flagged |= {int(q) for q in r.flagged_query}
    ok = np.array([q not in flagged for q in range(res * res)])
    assert ok.mean() > 0.9 and np.count_nonzero(orad.ravel()[ok]) > 10
    orad = orad.ravel()
    rel = np.abs(rad - orad) / np.maximum(np.abs(orad), 1e-300)
    rel[orad == 0] = np.abs(rad[orad == 0])
    assert np.max(rel[ok]) < 1e-4, np.max(rel[ok])
    _codes_agree(rgb[ok], orgb.reshape(-1, 3)[ok], orad[ok], 1.0)
