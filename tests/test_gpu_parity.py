"""GPU (CUDA path through the C-ABI) vs oracle parity — needs a B200.

Inputs are the seeded synthetic workloads; the oracle is the plain FP64 CPU transcription.  Every comparison
goes through tests/parity.py, which bounds each side's flagged fraction (2%), the tuples flagged on one side
only, and requires a minimum number of compared unflagged chains.
"""
import numpy as np
import pytest

import parity
from paper_2405_13409_b200 import workloads as W

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


def _gpu_solve(sp, torch, mesh, chain, ep, cfg=None, offsets=None, tri_ids=None, intensity=None):
    ctx = sp.Context(0, cfg)
    ctx.upload_mesh(mesh)
    e = torch.as_tensor(np.ascontiguousarray(ep), dtype=torch.float64, device="cuda")
    it = None if intensity is None else torch.as_tensor(intensity, dtype=torch.float64, device="cuda")
    off = None if offsets is None else torch.as_tensor(offsets.astype(np.int32), device="cuda")
    ids = None if tri_ids is None else torch.as_tensor(tri_ids.astype(np.int32), device="cuda")
    r = ctx.solve(chain, e, it, off, ids)
    out = r.to_numpy()
    out["report"] = r.report
    wl = ctx.last_worklist()
    out["worklist"] = (wl[0].cpu().numpy().view(np.uint32), wl[1].cpu().numpy().view(np.uint32).reshape(-1, len(chain)))
    ctx.close()
    return out


def _restrict(g, qs, k):
    """The GPU result of a full-size run restricted to the sampled queries qs (renumbered 0..len(qs)-1), with the
    sampled queries' work list as a CSR tuple list the oracle can solve (the identical tuples)."""
    remap = {int(q): i for i, q in enumerate(qs)}
    sel = np.isin(g["query"], qs)
    fsel = np.isin(g["flagged_query"], qs)
    pq, pt = g["worklist"]
    wsel = np.isin(pq, qs)
    wq = np.array([remap[int(q)] for q in pq[wsel]], np.uint32)
    wt = pt[wsel]
    order = np.argsort(wq, kind="stable")
    wq, wt = wq[order], wt[order]
    offsets = np.zeros(len(qs) + 1, np.uint32)
    np.add.at(offsets, wq + 1, 1)
    offsets = np.cumsum(offsets).astype(np.uint32)
    out = {"query": np.array([remap[int(q)] for q in g["query"][sel]], np.uint32), "tuple": g["tuple"][sel],
           "bary": g["bary"][sel], "per_query": g["per_query"][qs], "contribution": g["contribution"][sel],
           "residual": g["residual"][sel],
           "flagged_query": np.array([remap[int(q)] for q in g["flagged_query"][fsel]], np.uint32),
           "flagged_tuple": g["flagged_tuple"][fsel], "worklist": (wq, wt)}
    return out, offsets, np.ascontiguousarray(wt.reshape(-1)).astype(np.uint32), int(wsel.sum())


def test_sqrt_table_device_copy_matches_golden(sp, torch_cuda):
    """The kernels' constant-memory copy of the Eq. 20 sqrt surrogate (reading R8) is the golden table."""
    import os
    g = np.loadtxt(os.path.join(os.path.dirname(__file__), "golden", "sqrt_table.txt"))
    with sp.Context(0) as ctx:
        assert np.array_equal(sp.sqrt_table(ctx), g[:, :5])


def test_c1_patch_parity(orc, sp, torch_cuda):
    w = W.patch_c1()
    ro = orc.solve(w.mesh, "R", w.endpoints, cfg=orc.default_config(cull=0))
    g = _gpu_solve(sp, torch_cuda, w.mesh, "R", w.endpoints, cfg=sp.default_config(cull=0))
    parity.compare(ro, g, w.nqueries, min_compared=1, label="C1")
    assert g["report"]["n_pairs_in"] == w.mesh.ntris
    # culled run finds the same chains
    gc = _gpu_solve(sp, torch_cuda, w.mesh, "R", w.endpoints)
    parity.compare(ro, gc, w.nqueries, min_compared=1, label="C1 culled")


def test_flat_mirror_fixture_on_gpu(orc, sp, torch_cuda):
    """SURVEY §8(c) fixed point 1 on the GPU: the relabel decision (reading R1) picks e_2, a(., 1/3)
    is identically zero and the b fallback (c11) gives u = 1/2: x_1 = (0.5, 0, 0), (u, v) = (0.5, 1/3),
    J = (d_0 + d_1)^2."""
    pos = np.array([[-1, -1, 0], [2, -1, 0], [-1, 2, 0]], np.float32)
    nrm = np.tile([0, 0, 1], (3, 1)).astype(np.float32)
    mesh = W.Mesh(pos, nrm, np.array([[0, 1, 2]], np.uint32))
    ep = np.array([[[0, 0, 1], [1, 0, 1]]], float)
    g = _gpu_solve(sp, torch_cuda, mesh, "R", ep, cfg=sp.default_config(cull=0))
    assert g["query"].shape[0] == 1 and len(g["flagged_query"]) == 0
    assert np.allclose(g["bary"][0], [0.5, 1 / 3], atol=1e-9)
    assert np.isclose(1 / g["contribution"][0], (2 * np.sqrt(1.25)) ** 2, rtol=1e-8)
    ro = orc.solve(mesh, "R", ep, cfg=orc.default_config(cull=0))
    parity.compare(ro, g, 1, min_compared=1, label="S:520")


def test_random_interpolated_R(orc, sp, torch_cuda):
    rng = np.random.default_rng(12)
    mesh = W.random_triangles(rng, 300, 0.3, normal_tilt=0.3)
    Q = 24
    ep = np.zeros((Q, 2, 3))
    ep[:, 0] = rng.uniform(-1, 1, (Q, 3)) * [1, 1, 0.3] + [0, 0, 1.5]
    ep[:, 1] = rng.uniform(-1, 1, (Q, 3)) * [1, 1, 0.3] + [0, 0, 1.8]
    inten = rng.uniform(0.5, 2.0, Q)
    ro = orc.solve(mesh, "R", ep, intensity=inten, cfg=orc.default_config(cull=0))
    g = _gpu_solve(sp, torch_cuda, mesh, "R", ep, cfg=sp.default_config(cull=0), intensity=inten)
    parity.compare(ro, g, Q, min_compared=50, label="random R")
    # with the cull on both sides
    ro2 = orc.solve(mesh, "R", ep, intensity=inten)
    g2 = _gpu_solve(sp, torch_cuda, mesh, "R", ep, intensity=inten)
    parity.compare(ro2, g2, Q, min_compared=50, label="random R culled")
    # cull soundness: every oracle chain's (query, tuple) is in the GPU work list
    wl = set(zip(g2["worklist"][0].tolist(), g2["worklist"][1][:, 0].tolist()))
    assert all((int(q), int(t)) in wl for q, t in zip(ro2.query, ro2.tuple[:, 0]))


def test_explicit_tuple_list_and_edges(orc, sp, torch_cuda):
    w = W.patch_c1()
    ep = np.repeat(w.endpoints, 3, axis=0)
    ep[1, 1] += [0.05, -0.02, 0.0]
    # ragged CSR: every triangle for query 0, every third for query 1, 0 tuples for query 2
    ids0 = np.arange(0, 256, dtype=np.uint32)
    ids1 = np.arange(0, 256, 3, dtype=np.uint32)
    offsets = np.array([0, len(ids0), len(ids0) + len(ids1), len(ids0) + len(ids1)], np.uint32)
    tri_ids = np.concatenate([ids0, ids1])
    ro = orc.solve(w.mesh, "R", ep, offsets=offsets, tri_ids=tri_ids)
    g = _gpu_solve(sp, torch_cuda, w.mesh, "R", ep, offsets=offsets, tri_ids=tri_ids)
    parity.compare(ro, g, 3, min_compared=1, label="explicit list")
    assert g["per_query"][2] == 0.0
    assert g["report"]["n_pairs_in"] == len(tri_ids)


def test_empty_and_errors(sp, torch_cuda):
    torch = torch_cuda
    w = W.patch_c1()
    ctx = sp.Context(0)
    ctx.upload_mesh(w.mesh)
    r = ctx.solve("R", torch.zeros((0, 2, 3), dtype=torch.float64, device="cuda"))
    assert r.n_solutions == 0
    with pytest.raises(sp.SpolyError):
        ctx.solve("Q", torch.zeros((1, 2, 3), dtype=torch.float64, device="cuda"))
    # a triangle id out of range in an explicit tuple list: an error status, and the context stays usable
    ep = torch.as_tensor(w.endpoints, dtype=torch.float64, device="cuda")
    off = torch.as_tensor(np.array([0, 2], np.int32), device="cuda")
    bad_ids = torch.as_tensor(np.array([3, 100000], np.int32), device="cuda")
    with pytest.raises(sp.SpolyError):
        ctx.solve("R", ep, None, off, bad_ids)
    bad_off = torch.as_tensor(np.array([2, 1], np.int32), device="cuda")
    with pytest.raises(sp.SpolyError):
        ctx.solve("R", ep, None, bad_off, bad_ids)
    r = ctx.solve("R", ep)
    assert r.n_solutions >= 1
    bad = W.Mesh(np.zeros((3, 3), np.float32), np.tile([0, 0, 1], (3, 1)).astype(np.float32),
                 np.array([[0, 1, 2]], np.uint32))
    with pytest.raises(sp.SpolyError):
        ctx.upload_mesh(bad)
    ctx.close()


def test_c2_subset_parity(orc, sp, torch_cuda):
    """C2 glints mesh (100,352 tris), 24 light samples: cull + solve vs the oracle's own cull + solve."""
    w = W.glints_c2(res=256)
    sub = w.subset(np.arange(0, 65536, 65536 // 24)[:24])
    ro = orc.solve(sub.mesh, "R", sub.endpoints)
    g = _gpu_solve(sp, torch_cuda, sub.mesh, "R", sub.endpoints)
    parity.compare(ro, g, sub.nqueries, min_compared=1000, label="C2 subset")


def test_c2_full_size_sampled(orc, sp, torch_cuda):
    """Full C2 (65,536 queries) in the bench launch configuration; sampled queries re-solved by the oracle (its own
    cull), properties checked on every returned chain."""
    w = W.glints_c2(res=256)
    g = _gpu_solve(sp, torch_cuda, w.mesh, "R", w.endpoints)
    qs = np.sort(np.random.default_rng(99).choice(w.nqueries, 6, replace=False))
    sub = w.subset(qs)
    ro = orc.solve(sub.mesh, "R", sub.endpoints)
    gs, _, _, npairs = _restrict(g, qs, 1)
    parity.compare(ro, gs, len(qs), min_compared=100, gpu_pairs=npairs, label="C2 full sampled")
    # properties at full size: every returned vertex inside the triangle and specular (Eq. 3)
    assert np.all(g["residual"] < 1e-6)
    b = g["bary"]
    assert np.all(b[:, 0] >= -1e-9) and np.all(b[:, 1] >= -1e-9) and np.all(b.sum(1) <= 1 + 1e-9)
    assert abs(g["per_query"].sum() - g["contribution"].sum()) <= 1e-9 * abs(g["contribution"].sum())
    assert g["report"]["n_truncated"] == 0
    assert len(g["flagged_query"]) <= 0.02 * g["report"]["n_pairs_in"]


# ---------------------------------------------------------------- one-bounce refraction (T, Eq. 22)
def test_random_interpolated_T(orc, sp, torch_cuda):
    rng = np.random.default_rng(13)
    mesh = W.random_triangles(rng, 300, 0.3, normal_tilt=0.3)
    mesh.eta_front, mesh.eta_back = 1.0, 1.5
    Q = 24
    ep = np.zeros((Q, 2, 3))
    ep[:, 0] = rng.uniform(-1, 1, (Q, 3)) * [1, 1, 0.3] + [0, 0, 1.5]
    ep[:, 1] = rng.uniform(-1, 1, (Q, 3)) * [1, 1, 0.3] + [0, 0, -1.8]
    ep[Q // 2:] = ep[Q // 2:, ::-1]  # half the queries from below (both media orders)
    ro = orc.solve(mesh, "T", ep, cfg=orc.default_config(cull=0))
    g = _gpu_solve(sp, torch_cuda, mesh, "T", ep, cfg=sp.default_config(cull=0))
    parity.compare(ro, g, Q, min_compared=30, label="random T")
    ro2 = orc.solve(mesh, "T", ep)
    g2 = _gpu_solve(sp, torch_cuda, mesh, "T", ep)
    parity.compare(ro2, g2, Q, min_compared=30, label="random T culled")


def test_flat_interface_T(orc, sp, torch_cuda):
    pos = np.array([[-4, -4, 0], [6, -4, 0], [-4, 6, 0]], np.float32)
    nrm = np.tile([0, 0, 1], (3, 1)).astype(np.float32)
    mesh = W.Mesh(pos, nrm, np.array([[0, 1, 2]], np.uint32), 1.0, 1.33)
    rng = np.random.default_rng(3)
    ep = np.zeros((32, 2, 3))
    ep[:, 0] = np.c_[rng.uniform(-0.8, 0.8, (32, 2)), rng.uniform(0.5, 2, 32)]
    ep[:, 1] = np.c_[rng.uniform(-0.8, 0.8, (32, 2)), -rng.uniform(0.5, 2, 32)]
    ro = orc.solve(mesh, "T", ep, cfg=orc.default_config(cull=0))
    g = _gpu_solve(sp, torch_cuda, mesh, "T", ep, cfg=sp.default_config(cull=0))
    parity.compare(ro, g, 32, min_compared=32, label="flat interface")
    assert g["query"].shape[0] == 32  # exactly one refraction path per query


def test_c3_pool_subset_parity(orc, sp, torch_cuda):
    """C3 pool (199,712-tri water surface), 48 floor receivers: cull + solve vs the oracle's cull + solve."""
    w = W.pool_c3(res=512)
    sub = w.subset(np.linspace(0, w.nqueries - 1, 48).astype(np.int64))
    ro = orc.solve(sub.mesh, "T", sub.endpoints)
    g = _gpu_solve(sp, torch_cuda, sub.mesh, "T", sub.endpoints)
    parity.compare(ro, g, sub.nqueries, min_compared=20, label="C3 subset")
    assert np.all(g["residual"] < 1e-6)


def test_near_tangent_flags_at_folds_on_gpu(orc, sp, torch_cuda):
    """Fold configurations of a focusing interpolated-normal mirror (located by the oracle, pinned in
    test_oracle_pins_k2.py::test_near_tangent_flag_at_folds): the GPU flags NEAR_TANGENT there too, and the
    flag-aware parity holds on every configuration of the walk."""
    mesh = W.Mesh(*_concave_mirror_arrays())
    rng = np.random.default_rng(0)
    Q = 4000
    ep = np.zeros((Q, 2, 3))
    ep[:, 0] = rng.uniform(-2, 2, (Q, 3)) * [1, 1, 0] + [0, 0, 1] * rng.uniform(0.2, 3, (Q, 1))
    ep[:, 1] = rng.uniform(-2, 2, (Q, 3)) * [1, 1, 0] + [0, 0, 1] * rng.uniform(0.2, 3, (Q, 1))
    cfg = orc.default_config(cull=0)
    r = orc.solve(mesh, "R", ep, cfg=cfg)
    two = np.where(np.bincount(r.query, minlength=Q) == 2)[0]
    fold_eps = []
    for q in two[:6]:
        x0, x2 = ep[q]
        for trial in range(6):
            d = rng.normal(size=3)
            d /= np.linalg.norm(d)
            walk = np.array([[x0, x2 + s * d] for s in np.linspace(0, 1, 101)[1:]])
            rw = orc.solve(mesh, "R", walk, cfg=cfg)
            cnt = np.bincount(rw.query, minlength=len(walk))
            if cnt[0] != 2 or not np.any(cnt != 2):
                continue
            j = int(np.argmax(cnt != 2))
            if cnt[j] != 0:
                continue
            lo, hi = (j) / 100.0, (j + 1) / 100.0
            for _ in range(60):
                m = 0.5 * (lo + hi)
                rm = orc.solve(mesh, "R", np.array([[x0, x2 + m * d]]), cfg=cfg)
                if rm.n_solutions == 2:
                    lo = m
                else:
                    hi = m
            ra = orc.solve(mesh, "R", np.array([[x0, x2 + lo * d]]), cfg=cfg)
            if ra.n_solutions == 2 and np.max(np.abs(ra.bary[0] - ra.bary[1])) < 1e-3:
                fold_eps += [[x0, x2 + lo * d], [x0, x2 + hi * d], [x0, x2 + 0.5 * lo * d]]
            break
    assert len(fold_eps) >= 6
    fe = np.array(fold_eps)
    ro = orc.solve(mesh, "R", fe, cfg=cfg)
    g = _gpu_solve(sp, torch_cuda, mesh, "R", fe, cfg=sp.default_config(cull=0))
    gflag = {int(q): int(f) for q, f in zip(g["flagged_query"], g["flagged_flags"])}
    for i in range(0, len(fe), 3):
        assert gflag.get(i, 0) & sp.FLAG_NEAR_TANGENT and gflag.get(i + 1, 0) & sp.FLAG_NEAR_TANGENT, (i, gflag)
    # the flagged fraction here is 2/3 by construction: only the one-sided flags and the counts are held
    parity.compare(ro, g, len(fe), min_compared=1, max_flag_frac=1.0, label="folds")


def _concave_mirror_arrays(kappa=0.8):
    P = np.array([[-1, -1, 0], [1.2, -0.9, 0], [-0.8, 1.1, 0]], float)
    c = P.mean(0)
    N = np.array([np.array([0, 0, 1.0]) - kappa * (p - c) for p in P])
    N /= np.linalg.norm(N, axis=1)[:, None]
    return P.astype(np.float32), N.astype(np.float32), np.array([[0, 1, 2]], np.uint32)


# ---------------------------------------------------------------- two bounces (RR, TT; 100-piece scan)
def _planted_batch(chain, n, seed, size=0.15, face=False):
    from planted import planted_many
    cases = planted_many(seed, chain, n, size=size, face=face)
    pos, nrm, tri, eps = [], [], [], []
    for i, (m, ids, x0, xk1, bary) in enumerate(cases):
        pos.append(m.pos)
        nrm.append(m.nrm)
        tri.append(m.tri + 6 * i)
        eps.append([x0, xk1])
    mesh = W.Mesh(np.concatenate(pos), np.concatenate(nrm), np.concatenate(tri).astype(np.uint32),
                  cases[0][0].eta_front, cases[0][0].eta_back)
    ep = np.array(eps, float)
    rng = np.random.default_rng(seed + 1)
    offsets = [0]
    ids = []
    for i in range(len(cases)):
        tl = [(2 * i, 2 * i + 1)]
        while len(tl) < 3:  # two distinct decoy pairs from other configurations
            j, l = rng.integers(0, len(cases), 2)
            if (2 * int(j), 2 * int(l) + 1) not in tl:
                tl.append((2 * int(j), 2 * int(l) + 1))
        for a, b in tl:
            ids += [a, b]
        offsets.append(offsets[-1] + len(tl))
    return mesh, ep, np.array(offsets, np.uint32), np.array(ids, np.uint32), [c[4] for c in cases]


@pytest.mark.parametrize("chain", ["RR", "TT", "RT", "TR"])
def test_two_bounce_planted_parity(orc, sp, torch_cuda, chain):
    mesh, ep, off, ids, truth = _planted_batch(chain, 40, 61)
    ro = orc.solve(mesh, chain, ep, offsets=off, tri_ids=ids)
    g = _gpu_solve(sp, torch_cuda, mesh, chain, ep, offsets=off, tri_ids=ids)
    parity.compare(ro, g, len(ep), tol_bary=1e-4, min_compared=int(0.85 * len(ep)), label=f"planted {chain}")
    assert np.all(g["residual"] < 1e-6)
    # the planted chain is recovered on the GPU for most queries (100-piece scan misses are by design)
    hit = 0
    for qi, b in enumerate(truth):
        sel = g["query"] == qi
        if any(np.max(np.abs(x - b)) < 1e-6 for x in g["bary"][sel]):
            hit += 1
    assert hit >= int(0.9 * len(truth)), (hit, len(truth))


@pytest.mark.parametrize("chain", ["RR", "RT", "TR", "TT"])
def test_face_mode_planted_on_gpu(orc, sp, torch_cuda, chain):
    """Face-normal triangles (reading R22): 40/40 planted chains recovered unflagged on the GPU, parity
    with the oracle; RR on flat face mirrors has J = L^2 (unfolded path length)."""
    mesh, ep, off, ids, truth = _planted_batch(chain, 40, 171, face=True)
    ro = orc.solve(mesh, chain, ep, offsets=off, tri_ids=ids)
    g = _gpu_solve(sp, torch_cuda, mesh, chain, ep, offsets=off, tri_ids=ids)
    parity.compare(ro, g, len(ep), tol_bary=1e-4, min_compared=len(ep), label=f"face {chain}")
    for qi, b in enumerate(truth):
        sel = (g["query"] == qi) & (g["tuple"][:, 0] == 2 * qi) & (g["tuple"][:, 1] == 2 * qi + 1)
        d = [np.max(np.abs(x - b)) for x in g["bary"][sel]]
        assert d and min(d) < 1e-6, (qi, d)
        assert not np.any((g["flagged_query"] == qi) & (g["flagged_tuple"][:, 0] == 2 * qi)
                          & (g["flagged_tuple"][:, 1] == 2 * qi + 1))
        if chain == "RR":
            i = np.flatnonzero(sel)[int(np.argmin(d))]
            bb = g["bary"][i]
            P1 = mesh.pos[mesh.tri[2 * qi]].astype(float)
            P2 = mesh.pos[mesh.tri[2 * qi + 1]].astype(float)
            x1 = P1[0] + bb[0] * (P1[1] - P1[0]) + bb[1] * (P1[2] - P1[0])
            x2 = P2[0] + bb[2] * (P2[1] - P2[0]) + bb[3] * (P2[2] - P2[0])
            L = np.linalg.norm(x1 - ep[qi, 0]) + np.linalg.norm(x2 - x1) + np.linalg.norm(ep[qi, 1] - x2)
            assert abs((1 / g["contribution"][i]) / (L * L) - 1) < 1e-6


def test_two_bounce_tiles_vs_per_query_cull(sp, torch_cuda):
    """The tiled k=2 cull (32-query endpoint spheres + an exact per-query triangle-pair test) keeps every chain the
    per-query expansion finds: identical solution sets on a C4 subset (both culls are sound)."""
    w = W.sphere_c4(res=32, level=4)
    a = _gpu_solve(sp, torch_cuda, w.mesh, "TT", w.endpoints, cfg=sp.default_config(k2_tiles=0))
    b = _gpu_solve(sp, torch_cuda, w.mesh, "TT", w.endpoints, cfg=sp.default_config(k2_tiles=1))
    key = lambda g: sorted(zip(g["query"].tolist(), map(tuple, g["tuple"].tolist()), map(tuple, np.round(g["bary"], 12).tolist())))
    assert a["report"]["n_admissible"] > 100
    assert key(a) == key(b)
    assert np.array_equal(a["per_query"], b["per_query"])


@pytest.mark.parametrize("chain", ["RR", "TT"])
def test_two_bounce_cull_sound_on_planted(orc, sp, torch_cuda, chain):
    """GPU pair cull (no tuple list) keeps every planted pair and the solve recovers the planted chains."""
    mesh, ep, off, ids, truth = _planted_batch(chain, 12, 71)
    g = _gpu_solve(sp, torch_cuda, mesh, chain, ep)
    pq, pt = g["worklist"]
    for qi in range(len(ep)):
        assert np.any((pq == qi) & (pt[:, 0] == 2 * qi) & (pt[:, 1] == 2 * qi + 1)), qi
    ro = orc.solve(mesh, chain, ep)  # the oracle's own cull
    parity.compare(ro, g, len(ep), tol_bary=1e-4, min_compared=int(0.8 * len(ep)), label=f"cull {chain}")


def test_rr_mirrors_parity(orc, sp, torch_cuda):
    """C5 RR variant (two facing bumpy mirrors): GPU pair cull + solve vs the oracle's cull + solve."""
    w = W.mirrors_rr(res=8, quads=16)
    sub = w.subset(np.arange(0, 64, 8))
    ro = orc.solve(sub.mesh, "RR", sub.endpoints)
    g = _gpu_solve(sp, torch_cuda, sub.mesh, "RR", sub.endpoints)
    parity.compare(ro, g, sub.nqueries, tol_bary=1e-4, min_compared=10, label="RR mirrors")
    assert g["report"]["n_pairs_in"] >= ro.report["pairs_in"]


def test_tt_sphere_parity(orc, sp, torch_cuda):
    """C4-shaped dielectric icosphere (level 2, 320 tris), TT through it: GPU cull + solve vs the oracle."""
    w = W.sphere_c4(res=8, level=2)
    sub = w.subset([18, 19, 20, 27, 28, 29, 36, 37])
    ro = orc.solve(sub.mesh, "TT", sub.endpoints)
    g = _gpu_solve(sp, torch_cuda, sub.mesh, "TT", sub.endpoints)
    parity.compare(ro, g, sub.nqueries, tol_bary=1e-4, min_compared=8, label="TT sphere L2")


def test_tt_big_order_branch(orc, sp, torch_cuda):
    """Level-1 icosphere (80 large triangles): about half the TT tuples keep a numerical Bezout order n > 32
    (reading R6), which the scan evaluates with the shared-memory elimination; the report's counter proves the
    branch ran, and the parity holds on those tuples too."""
    w = W.sphere_c4(res=8, level=1)
    sub = w.subset([18, 19, 27, 28, 36, 37])
    ro = orc.solve(sub.mesh, "TT", sub.endpoints)
    g = _gpu_solve(sp, torch_cuda, sub.mesh, "TT", sub.endpoints)
    assert g["report"]["n_big_scan"] > 0, g["report"]
    parity.compare(ro, g, sub.nqueries, tol_bary=1e-4, min_compared=4, label="TT sphere L1 (n > 32)")


@pytest.mark.parametrize("name,make,nsample", [("C4", lambda: W.sphere_c4(res=128, level=4), 8),
                                               ("C5", lambda: W.shell_c5(res=128, level=3), 8)])
def test_two_bounce_full_size_sampled(orc, sp, torch_cuda, name, make, nsample):
    """Full-size k=2 frames in the bench launch configuration (C4: 16,384 receivers x 5,120-tri sphere, TT; C5 shell
    at the bench's 16,384 receivers): sampled receivers re-solved by the oracle on the identical tuples (the GPU's
    refined pair list of those receivers); every returned chain satisfies Eq. 3 and the domain, and no per-tuple
    capacity was hit."""
    w = make()
    g = _gpu_solve(sp, torch_cuda, w.mesh, "TT", w.endpoints)
    rep = g["report"]
    assert rep["n_admissible"] > 1000 and rep["n_truncated"] == 0
    assert len(g["flagged_query"]) <= 0.02 * rep["n_pairs_in"], (len(g["flagged_query"]), rep["n_pairs_in"])
    # sampled receivers: those with chains, spread over the frame
    with_sol = np.unique(g["query"])
    qs = np.sort(np.random.default_rng(5).choice(with_sol, nsample, replace=False))
    gs, off, ids, npairs = _restrict(g, qs, 2)
    sub = w.subset(qs)
    ro = orc.solve(sub.mesh, "TT", sub.endpoints, offsets=off, tri_ids=ids)
    parity.compare(ro, gs, len(qs), tol_bary=1e-4, min_compared=nsample, gpu_pairs=npairs, label=f"{name} full sampled")
    assert np.all(g["residual"] < 1e-6)
    b = g["bary"]
    for c in (0, 2):
        assert np.all(b[:, c] >= -1e-9) and np.all(b[:, c + 1] >= -1e-9) and np.all(b[:, c] + b[:, c + 1] <= 1 + 1e-9)


def test_c3_full_size_sampled(orc, sp, torch_cuda):
    """Full C3 (262,144 receivers x 199,712 tris, T) in the bench launch configuration; sampled receivers
    re-solved by the oracle; properties checked on every returned chain."""
    w = W.pool_c3(res=512)
    g = _gpu_solve(sp, torch_cuda, w.mesh, "T", w.endpoints)
    qs = np.sort(np.random.default_rng(7).choice(w.nqueries, 24, replace=False))
    sub = w.subset(qs)
    ro = orc.solve(sub.mesh, "T", sub.endpoints)
    gs, _, _, npairs = _restrict(g, qs, 1)
    parity.compare(ro, gs, len(qs), min_compared=12, gpu_pairs=npairs, label="C3 full sampled")
    assert np.all(g["residual"] < 1e-6)
    b = g["bary"]
    assert np.all(b[:, 0] >= -1e-9) and np.all(b[:, 1] >= -1e-9) and np.all(b.sum(1) <= 1 + 1e-9)
    assert len(g["flagged_query"]) <= 0.02 * g["report"]["n_pairs_in"]


def test_determinism_bit_identical(sp, torch_cuda):
    """Two solves of the same inputs give bit-identical outputs."""
    w = W.glints_c2(res=32)
    a = _gpu_solve(sp, torch_cuda, w.mesh, "R", w.endpoints)
    b = _gpu_solve(sp, torch_cuda, w.mesh, "R", w.endpoints)
    for k in ("query", "tuple", "bary", "contribution", "per_query", "flagged_query"):
        assert np.array_equal(a[k], b[k]), k


@pytest.mark.parametrize("chain,make", [("R", lambda: W.glints_c2(res=48)), ("T", lambda: W.pool_c3(res=64)),
                                        ("TT", lambda: W.shell_c5(res=8))])
def test_counting_order_equals_key_sort(sp, torch_cuda, monkeypatch, chain, make):
    """The counting order (slot masks + scanned pair counts + scatter) writes the solutions in exactly the
    order of the (pair << 6 | slot) key sort it replaces: every output array is bit-identical."""
    w = make()
    monkeypatch.setenv("SPOLY_SORT_ORDER", "0")
    a = _gpu_solve(sp, torch_cuda, w.mesh, chain, w.endpoints, intensity=w.intensity)
    monkeypatch.setenv("SPOLY_SORT_ORDER", "1")
    b = _gpu_solve(sp, torch_cuda, w.mesh, chain, w.endpoints, intensity=w.intensity)
    assert a["report"]["n_admissible"] > 0
    for k in ("query", "tuple", "bary", "contribution", "residual", "flags", "per_query", "flagged_query",
              "flagged_flags"):
        assert np.array_equal(a[k], b[k]), k


@pytest.mark.parametrize("chain,make", [("RR", lambda: W.mirrors_rr(res=16, quads=16)),
                                        ("TT", lambda: W.shell_c5(res=16))])
def test_two_bounce_query_chunking_identical(sp, torch_cuda, chain, make):
    """cfg.max_pairs small enough that the k=2 cull runs in many query chunks (whole tiles of 32 Morton-sorted
    queries): the work list, solutions and per-query sums are bit-identical to the single-chunk run (chunks append
    in sorted-query order)."""
    w = make()
    a = _gpu_solve(sp, torch_cuda, w.mesh, chain, w.endpoints)
    # a budget of a third of the whole frame's triangle-pair frontier: several chunks, each within budget
    budget = a["report"]["n_pairs_coarse"] // 3 + 1
    b = _gpu_solve(sp, torch_cuda, w.mesh, chain, w.endpoints, cfg=sp.default_config(max_pairs=budget))
    assert b["report"]["n_pairs_coarse"] == a["report"]["n_pairs_coarse"]
    assert a["report"]["n_pairs_in"] == b["report"]["n_pairs_in"] > 0
    assert np.array_equal(a["worklist"][0], b["worklist"][0])
    assert np.array_equal(a["worklist"][1], b["worklist"][1])
    for k in ("query", "tuple", "bary", "contribution", "per_query", "flagged_query", "flagged_tuple"):
        assert np.array_equal(a[k], b[k]), k


# ---------------------------------------------------------------- visibility
def _blockers(rng, n, center, spread, size):
    P = []
    for _ in range(n):
        c = np.asarray(center) + rng.uniform(-1, 1, 3) * spread
        P.append(c + rng.normal(size=(3, 3)) * size)
    P = np.concatenate(P).astype(np.float32)
    return W.Mesh(P, np.tile([0, 0, 1], (len(P), 1)).astype(np.float32), np.arange(len(P), dtype=np.uint32).reshape(-1, 3))


@pytest.mark.parametrize("chain", ["R", "RR", "TT"])
def test_visibility_parity(orc, sp, torch_cuda, chain):
    """cfg.visibility = 1 with occluders floating over the chains (and the specular mesh occluding itself): the GPU's
    AABB-hierarchy segment test drops exactly the chains the oracle's brute force drops (same counts, same survivors,
    same per-query sums)."""
    rng = np.random.default_rng(201)
    if chain == "R":
        w = W.glints_c2(res=256)
        sub = w.subset(np.arange(0, 65536, 65536 // 16)[:16])
        mesh, ep, off, ids = sub.mesh, sub.endpoints, None, None
        occ = _blockers(rng, 400, (0.0, 0.0, 0.4), np.array([1.0, 1.0, 0.3]), 0.03)
    else:
        mesh, ep, off, ids, _ = _planted_batch(chain, 30, 211)
        # blockers around the segments of the planted chains
        pts = []
        for q in range(len(ep)):
            a, b = ep[q]
            pts.append(a + rng.uniform(0.2, 0.8) * (b - a))
        occ = _blockers(rng, 1, (0, 0, 0), np.zeros(3), 0.0)
        P = np.concatenate([p + rng.normal(size=(3, 3)) * 0.08 for p in pts]).astype(np.float32)
        occ = W.Mesh(P, np.tile([0, 0, 1], (len(P), 1)).astype(np.float32), np.arange(len(P), dtype=np.uint32).reshape(-1, 3))
    ro = orc.solve(mesh, chain, ep, offsets=off, tri_ids=ids, cfg=orc.default_config(visibility=1), occluders=occ)
    ctx = sp.Context(0, sp.default_config(visibility=1))
    ctx.upload_mesh(mesh)
    ctx.upload_occluders(occ)
    torch = torch_cuda
    e = torch.as_tensor(np.ascontiguousarray(ep), dtype=torch.float64, device="cuda")
    o = None if off is None else torch.as_tensor(off.astype(np.int32), device="cuda")
    t = None if ids is None else torch.as_tensor(ids.astype(np.int32), device="cuda")
    r = ctx.solve(chain, e, None, o, t)
    g = r.to_numpy()
    g["report"] = r.report
    wl = ctx.last_worklist()
    g["worklist"] = (wl[0].cpu().numpy().view(np.uint32), wl[1].cpu().numpy().view(np.uint32).reshape(-1, len(chain)))
    ctx.close()
    assert ro.report["rej_visibility"] > 0
    assert g["report"]["n_rej_visibility"] == ro.report["rej_visibility"], (g["report"]["n_rej_visibility"],
                                                                             ro.report["rej_visibility"])
    parity.compare(ro, g, len(ep), tol_bary=1e-5 if len(chain) == 1 else 1e-4, min_compared=5 if len(chain) == 1 else 3,
                   label=f"visibility {chain}")


@pytest.mark.parametrize("chain,make", [("TT", lambda: W.sphere_c4(res=32, level=4)),
                                        ("TT", lambda: W.shell_c5(res=32, level=3)),
                                        ("RR", lambda: W.mirrors_rr(res=16, quads=32))])
def test_scan_restriction_keeps_every_chain(sp, torch_cuda, chain, make):
    """Reading R25: skipping the scan pieces outside the v-range of T_1's surviving cull cells changes no admissible
    chain (same roots on the kept pieces, same bisection, same polish): the solution arrays are bit-identical to the
    full 100-piece scan, and fewer determinants are evaluated."""
    w = make()
    a = _gpu_solve(sp, torch_cuda, w.mesh, chain, w.endpoints, cfg=sp.default_config(scan_restrict=0))
    b = _gpu_solve(sp, torch_cuda, w.mesh, chain, w.endpoints, cfg=sp.default_config(scan_restrict=1))
    assert a["report"]["n_admissible"] > 0
    for k in ("query", "tuple", "bary", "contribution", "residual", "per_query"):
        assert np.array_equal(a[k], b[k]), k
    assert b["report"]["alg_kflop"] < a["report"]["alg_kflop"]
