"""GPU (CUDA path through the C-ABI) vs oracle parity — needs a B200.

Inputs are the seeded synthetic workloads; the oracle is the plain FP64 CPU transcription.
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


def test_c1_patch_parity(orc, sp, torch_cuda):
    w = W.patch_c1()
    ro = orc.solve(w.mesh, "R", w.endpoints, cfg=orc.default_config(cull=0))
    g = _gpu_solve(sp, torch_cuda, w.mesh, "R", w.endpoints, cfg=sp.default_config(cull=0))
    st = parity.compare(ro, g, w.nqueries)
    assert g["report"]["n_pairs_in"] == w.mesh.ntris
    assert st["compared_solutions"] >= 1
    # culled run finds the same chains
    gc = _gpu_solve(sp, torch_cuda, w.mesh, "R", w.endpoints)
    parity.compare(ro, gc, w.nqueries)


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
    st = parity.compare(ro, g, Q)
    assert st["compared_solutions"] > 50, st
    # with the cull on both sides
    ro2 = orc.solve(mesh, "R", ep, intensity=inten)
    g2 = _gpu_solve(sp, torch_cuda, mesh, "R", ep, intensity=inten)
    parity.compare(ro2, g2, Q)
    # cull soundness: every oracle chain's (query, tuple) is in the GPU work list
    wl = set(zip(g2["worklist"][0].tolist(), g2["worklist"][1][:, 0].tolist()))
    assert all((int(q), int(t)) in wl for q, t in zip(ro2.query, ro2.tuple[:, 0]))


def test_explicit_tuple_list_and_edges(orc, sp, torch_cuda):
    w = W.patch_c1()
    ep = np.repeat(w.endpoints, 3, axis=0)
    ep[1, 1] += [0.05, -0.02, 0.0]
    # ragged CSR: 0 tuples for query 2
    ids = np.arange(0, 256, 3, dtype=np.uint32)
    offsets = np.array([0, len(ids), 2 * len(ids), 2 * len(ids)], np.uint32)
    tri_ids = np.concatenate([ids, ids])
    ro = orc.solve(w.mesh, "R", ep, offsets=offsets, tri_ids=tri_ids)
    g = _gpu_solve(sp, torch_cuda, w.mesh, "R", ep, offsets=offsets, tri_ids=tri_ids)
    parity.compare(ro, g, 3)
    assert g["per_query"][2] == 0.0
    assert g["report"]["n_pairs_in"] == 2 * len(ids)


def test_empty_and_errors(sp, torch_cuda):
    torch = torch_cuda
    w = W.patch_c1()
    ctx = sp.Context(0)
    ctx.upload_mesh(w.mesh)
    r = ctx.solve("R", torch.zeros((0, 2, 3), dtype=torch.float64, device="cuda"))
    assert r.n_solutions == 0
    with pytest.raises(sp.SpolyError):
        ctx.solve("Q", torch.zeros((1, 2, 3), dtype=torch.float64, device="cuda"))
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
    st = parity.compare(ro, g, sub.nqueries)
    assert st["compared_solutions"] > 1000, st
    assert st["flagged_tuples"] <= 0.01 * g["report"]["n_pairs_in"], st


def test_c2_full_size_sampled(orc, sp, torch_cuda):
    """Full C2 (65,536 queries) in the bench launch configuration; sampled queries re-solved by the oracle."""
    w = W.glints_c2(res=256)
    g = _gpu_solve(sp, torch_cuda, w.mesh, "R", w.endpoints)
    rng = np.random.default_rng(99)
    qs = np.sort(rng.choice(w.nqueries, 6, replace=False))
    sub = w.subset(qs)
    ro = orc.solve(sub.mesh, "R", sub.endpoints)
    # restrict the GPU result to the sampled queries, renumbered 0..5
    sel = np.isin(g["query"], qs)
    remap = {int(q): i for i, q in enumerate(qs)}
    gs = {"query": np.array([remap[int(q)] for q in g["query"][sel]], np.uint32), "tuple": g["tuple"][sel],
          "bary": g["bary"][sel], "per_query": g["per_query"][qs]}
    fsel = np.isin(g["flagged_query"], qs)
    gs["flagged_query"] = np.array([remap[int(q)] for q in g["flagged_query"][fsel]], np.uint32)
    gs["flagged_tuple"] = g["flagged_tuple"][fsel]
    gs["contribution"] = g["contribution"][sel]
    st = parity.compare(ro, gs, len(qs))
    assert st["compared_solutions"] > 100
    # properties at full size: every returned vertex inside the triangle and specular (Eq. 3)
    assert np.all(g["residual"] < 1e-6)
    b = g["bary"]
    assert np.all(b[:, 0] >= -1e-9) and np.all(b[:, 1] >= -1e-9) and np.all(b.sum(1) <= 1 + 1e-9)
    assert abs(g["per_query"].sum() - g["contribution"].sum()) <= 1e-9 * abs(g["contribution"].sum())


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
    st = parity.compare(ro, g, Q)
    assert st["compared_solutions"] > 30, st
    ro2 = orc.solve(mesh, "T", ep)
    g2 = _gpu_solve(sp, torch_cuda, mesh, "T", ep)
    parity.compare(ro2, g2, Q)


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
    parity.compare(ro, g, 32)
    assert g["query"].shape[0] == 32  # exactly one refraction path per query


def test_c3_pool_subset_parity(orc, sp, torch_cuda):
    """C3 pool (199,712-tri water surface), 48 floor receivers: cull + solve vs the oracle's cull + solve."""
    w = W.pool_c3(res=512)
    sub = w.subset(np.linspace(0, w.nqueries - 1, 48).astype(np.int64))
    ro = orc.solve(sub.mesh, "T", sub.endpoints)
    g = _gpu_solve(sp, torch_cuda, sub.mesh, "T", sub.endpoints)
    st = parity.compare(ro, g, sub.nqueries)
    assert st["compared_solutions"] >= 20, st
    assert np.all(g["residual"] < 1e-6)


# ---------------------------------------------------------------- two bounces (RR, TT; 100-piece scan)
def _planted_batch(chain, n, seed, size=0.15):
    from planted import planted_many
    cases = planted_many(seed, chain, n, size=size)
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
        for _ in range(2):  # decoy pairs from other configurations
            j, l = rng.integers(0, len(cases), 2)
            tl.append((2 * int(j), 2 * int(l) + 1))
        for a, b in tl:
            ids += [a, b]
        offsets.append(offsets[-1] + len(tl))
    return mesh, ep, np.array(offsets, np.uint32), np.array(ids, np.uint32), [c[4] for c in cases]


@pytest.mark.parametrize("chain", ["RR", "TT", "RT", "TR"])
def test_two_bounce_planted_parity(orc, sp, torch_cuda, chain):
    mesh, ep, off, ids, truth = _planted_batch(chain, 16 if chain[0] == "R" else 8, 61)
    ro = orc.solve(mesh, chain, ep, offsets=off, tri_ids=ids)
    g = _gpu_solve(sp, torch_cuda, mesh, chain, ep, offsets=off, tri_ids=ids)
    st = parity.compare(ro, g, len(ep), tol_bary=1e-4)
    assert st["compared_solutions"] >= len(ep) // 2, st
    assert np.all(g["residual"] < 1e-6)
    # the planted chain is recovered on the GPU for most queries (100-piece scan misses are by design)
    hit = 0
    for qi, b in enumerate(truth):
        sel = g["query"] == qi
        if any(np.max(np.abs(x - b)) < 1e-6 for x in g["bary"][sel]):
            hit += 1
    assert hit >= int(0.85 * len(truth)), (hit, len(truth))


@pytest.mark.parametrize("chain", ["RR", "TT"])
def test_two_bounce_cull_sound_on_planted(orc, sp, torch_cuda, chain):
    """GPU pair cull (no tuple list) keeps every planted pair and the solve recovers the planted chains."""
    mesh, ep, off, ids, truth = _planted_batch(chain, 12, 71)
    g = _gpu_solve(sp, torch_cuda, mesh, chain, ep)
    pq, pt = g["worklist"]
    for qi in range(len(ep)):
        assert np.any((pq == qi) & (pt[:, 0] == 2 * qi) & (pt[:, 1] == 2 * qi + 1)), qi
    ro = orc.solve(mesh, chain, ep)  # the oracle's own cull
    parity.compare(ro, g, len(ep), tol_bary=1e-4)


def test_rr_mirrors_parity(orc, sp, torch_cuda):
    """C5 RR variant (two facing bumpy mirrors): GPU pair cull + solve vs the oracle's cull + solve."""
    w = W.mirrors_rr(res=8, quads=16)
    sub = w.subset(np.arange(0, 64, 8))
    ro = orc.solve(sub.mesh, "RR", sub.endpoints)
    g = _gpu_solve(sp, torch_cuda, sub.mesh, "RR", sub.endpoints)
    st = parity.compare(ro, g, sub.nqueries, tol_bary=1e-4)
    assert st["compared_solutions"] >= 10, st
    assert g["report"]["n_pairs_in"] >= ro.report["pairs_in"]


def test_tt_sphere_parity(orc, sp, torch_cuda):
    """C4-shaped dielectric icosphere (level 2, 320 tris), TT through it: GPU cull + solve vs the oracle."""
    w = W.sphere_c4(res=4, level=2)
    sub = w.subset([5, 6])
    ro = orc.solve(sub.mesh, "TT", sub.endpoints)
    g = _gpu_solve(sp, torch_cuda, sub.mesh, "TT", sub.endpoints)
    parity.compare(ro, g, sub.nqueries, tol_bary=1e-4)


def test_c3_full_size_sampled(orc, sp, torch_cuda):
    """Full C3 (262,144 receivers x 199,712 tris, T) in the bench launch configuration; sampled receivers
    re-solved by the oracle; properties checked on every returned chain."""
    w = W.pool_c3(res=512)
    g = _gpu_solve(sp, torch_cuda, w.mesh, "T", w.endpoints)
    qs = np.sort(np.random.default_rng(7).choice(w.nqueries, 24, replace=False))
    sub = w.subset(qs)
    ro = orc.solve(sub.mesh, "T", sub.endpoints)
    sel = np.isin(g["query"], qs)
    remap = {int(q): i for i, q in enumerate(qs)}
    fsel = np.isin(g["flagged_query"], qs)
    gs = {"query": np.array([remap[int(q)] for q in g["query"][sel]], np.uint32), "tuple": g["tuple"][sel],
          "bary": g["bary"][sel], "per_query": g["per_query"][qs], "contribution": g["contribution"][sel],
          "flagged_query": np.array([remap[int(q)] for q in g["flagged_query"][fsel]], np.uint32),
          "flagged_tuple": g["flagged_tuple"][fsel]}
    st = parity.compare(ro, gs, len(qs))
    assert st["compared_solutions"] >= 12
    assert np.all(g["residual"] < 1e-6)
    b = g["bary"]
    assert np.all(b[:, 0] >= -1e-9) and np.all(b[:, 1] >= -1e-9) and np.all(b.sum(1) <= 1 + 1e-9)


def test_determinism_bit_identical(sp, torch_cuda):
    """deterministic=1: two solves of the same inputs give bit-identical outputs."""
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


@pytest.mark.parametrize("chain,make", [("RR", lambda: W.mirrors_rr(res=8, quads=16)),
                                        ("TT", lambda: W.shell_c5(res=8))])
def test_two_bounce_query_chunking_identical(sp, torch_cuda, chain, make):
    """cfg.max_pairs small enough that the k=2 cull runs in many query chunks: the work list, solutions and
    per-query sums are bit-identical to the single-chunk run (chunks append in query order)."""
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
