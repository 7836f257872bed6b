"""Oracle pins of the glossy extension (reading R28) and of the deterministic splat
renderer (SPEC S:661-669 cmd_render).  No GPU.

- the normal offset is pinned by its frame properties (tangential, components p along e1 and q along g^ x e1) and by
  the zero-offset identity;
- a glossy solve is a specular solve of the perturbed surface: brute-force shooting on that surface (an independent
  finder) must find the same chains;
- the renderer is pinned by the image-source construction of a flat-mirror caustic (lit mask IoU = 1, radiance
  albedo/pi * I / L^2 with L the unfolded path length) and by the gamma-2.2 code of known values.
"""
import numpy as np
import pytest

import bruteforce
from paper_2405_13409_b200.workloads import (MIRROR_LIGHT, beckmann_slopes, mirror_caustic, patch_c1,
                                              random_triangles)


def _match(a, b, tol):
    if len(a) != len(b):
        return False
    used = set()
    for x in a:
        d = [np.max(np.abs(np.asarray(x) - np.asarray(y))) if j not in used else np.inf for j, y in enumerate(b)]
        j = int(np.argmin(d)) if d else -1
        if j < 0 or d[j] > tol:
            return False
        used.add(j)
    return True


def test_zero_offset_is_identity(orc):
    w = patch_c1()
    m = orc.perturb_normals(w.mesh, np.zeros((w.mesh.ntris, 2)))
    tri = w.mesh.tri.astype(np.int64)
    assert np.array_equal(m.nrm.reshape(-1, 3, 3), w.mesh.nrm[tri])
    assert np.array_equal(m.pos.reshape(-1, 3, 3), w.mesh.pos[tri])
    a = orc.solve(w.mesh, "R", w.endpoints)
    b = orc.solve(m, "R", w.endpoints)
    assert a.n_solutions >= 1
    assert np.array_equal(a.tuple, b.tuple) and np.array_equal(a.bary, b.bary)
    assert np.array_equal(a.per_query, b.per_query)


def test_offset_frame_properties(orc):
    # reading R28: the offset lies in the triangle plane, its component along e1 is p and along g^ x e1 is q
    rng = np.random.default_rng(41)
    mesh = random_triangles(rng, 60, 0.4, normal_tilt=0.3)
    sl = beckmann_slopes(7, 1, mesh.ntris, 0.3)[0]
    m = orc.perturb_normals(mesh, sl)
    tri = mesh.tri.astype(np.int64)
    P = mesh.pos[tri].astype(np.float64)
    d = m.nrm.reshape(-1, 3, 3).astype(np.float64) - mesh.nrm[tri].astype(np.float64)
    e1, e2 = P[:, 1] - P[:, 0], P[:, 2] - P[:, 0]
    g = np.cross(e1, e2)
    for t in range(mesh.ntris):
        gh = g[t] / np.linalg.norm(g[t])
        ex = e1[t] / np.linalg.norm(e1[t])
        ey = np.cross(gh, ex)
        assert np.isclose(np.dot(ex, ey), 0, atol=1e-12) and np.isclose(np.linalg.det([ex, ey, gh]), 1.0)
        for j in range(3):  # the same offset on all three vertices (fl32 rounding of n + offset: 1e-7)
            assert abs(np.dot(d[t, j], gh)) < 2e-7
            assert abs(np.dot(d[t, j], ex) - sl[t, 0]) < 2e-7
            assert abs(np.dot(d[t, j], ey) - sl[t, 1]) < 2e-7


def test_offset_tilts_flat_normal_by_slope_angle(orc):
    # a face-normal triangle: the microfacet normal makes angle atan(sqrt(p^2 + q^2)) with the face normal
    pos = np.array([[0, 0, 0], [1, 0.2, 0.1], [0.1, 1, -0.2]], np.float32)
    g = np.cross(pos[1].astype(float) - pos[0], pos[2].astype(float) - pos[0])
    nrm = np.tile(g / np.linalg.norm(g), (3, 1)).astype(np.float32)
    from paper_2405_13409_b200.workloads import Mesh
    mesh = Mesh(pos, nrm, np.array([[0, 1, 2]], np.uint32))
    for p, q in [(0.3, 0.0), (0.0, -0.4), (0.2, 0.25)]:
        m = orc.perturb_normals(mesh, np.array([[p, q]]))
        n2 = m.nrm[0].astype(np.float64)
        ang = np.arccos(np.dot(n2, nrm[0]) / np.linalg.norm(n2) / np.linalg.norm(nrm[0]))
        assert np.isclose(ang, np.arctan(np.hypot(p, q)), atol=1e-6)


@pytest.mark.parametrize("chain", ["R", "T"])
def test_glossy_solve_matches_bruteforce(orc, chain):
    # PAPER.md:859 "the problem reduces to pure specular situations": shoot on the perturbed surface
    rng = np.random.default_rng(12 if chain == "R" else 22)
    mesh = random_triangles(rng, 60, 0.35, normal_tilt=0.25)
    mesh.eta_front, mesh.eta_back = 1.0, 1.5
    m = orc.perturb_normals(mesh, beckmann_slopes(3, 1, mesh.ntris, 0.2)[0])
    eps = [[[0.1, -0.3, 1.5], [0.4, 0.6, 1.2]], [[-0.6, 0.2, 0.9], [0.7, -0.1, 2.0]]]
    if chain == "T":
        eps = [[[0.1, -0.3, 1.5], [0.4, 0.6, -1.2]], [[-0.6, 0.2, -0.9], [0.7, -0.1, 2.0]],
               [[0.3, 0.2, 1.9], [-0.2, -0.1, -1.0]]]
    ep = np.array(eps, float)
    r = orc.solve(m, chain, ep, cfg=orc.default_config(cull=0))
    total = 0
    for qi in range(len(ep)):
        fl = {int(t) for q, t in zip(r.flagged_query, r.flagged_tuple[:, 0]) if q == qi}
        for t in range(mesh.ntris):
            if t in fl:
                continue
            bf = bruteforce.brute_force(chain, m, [t], ep[qi, 0], ep[qi, 1], grid=160, eta_front=m.eta_front,
                                        eta_back=m.eta_back)
            mine = [r.bary[i] for i in range(r.n_solutions) if r.query[i] == qi and r.tuple[i, 0] == t]
            assert _match(mine, bf, 1e-6), (qi, t, mine, bf)
            total += len(bf)
    assert total >= 3


def image_source_mask(res, half=1.5):
    """lit receivers of the mirror_caustic fixture by the image-source construction: the segment from x_0 to the
    light mirrored in z = 1 crosses the mirror triangle; returns (lit, unfolded length, margin)"""
    w = mirror_caustic(res, half)
    P = w.mesh.pos.astype(np.float64)
    Lp = np.array(MIRROR_LIGHT, float)
    Lp[2] = 2.0 - Lp[2]
    x0 = w.endpoints[:, 0]
    X = x0 + (1.0 / Lp[2]) * (Lp - x0)  # crossing of z = 1
    # barycentrics of X in the triangle (2-D, z = 1)
    a, b, c = P[0, :2], P[1, :2], P[2, :2]
    M = np.array([b - a, c - a]).T
    uv = np.linalg.solve(M, (X[:, :2] - a).T).T
    bar = np.stack([1 - uv[:, 0] - uv[:, 1], uv[:, 0], uv[:, 1]], 1)
    lit = np.all(bar > 0, axis=1)
    return w, lit, np.linalg.norm(Lp - x0, axis=1), np.min(np.abs(bar), axis=1)


def test_render_mirror_caustic_image_source(orc):
    # lit pixels exactly where the image-source construction predicts (mask IoU = 1); radiance of a lit
    # pixel = albedo / pi * I / L^2 (a flat mirror's J is the squared unfolded length)
    res = 64
    w, lit, L, margin = image_source_mask(res)
    rad, rgb, _ = orc.render(w.mesh, "R", w.endpoints, res, res, intensity=w.intensity, albedo=0.8)
    rad = rad.ravel()
    clear = margin > 1e-6
    got = rad > 0
    inter = np.sum(got & lit & clear)
    union = np.sum((got | lit) & clear)
    assert lit.sum() > 50 and inter == union, (inter, union)
    assert np.allclose(rad[lit & clear], 0.8 / np.pi / L[lit & clear] ** 2, rtol=1e-8)


def test_tonemap_codes(orc):
    v = np.array([0.0, -1.0, 1.0, 5.0, 0.5 ** 2.2, (10.0 / 255.0) ** 2.2])
    c = orc.tonemap_srgb(v)[:, 0]
    assert list(c) == [0, 0, 255, 255, 128, 10]
    assert np.array_equal(orc.tonemap_srgb(np.array([0.25]), exposure=4.0), [[255, 255, 255]])


def test_render_samples_average(orc):
    # S identical offset samples render the single-sample image; zero offsets render the specular image
    w = mirror_caustic(24)
    sl = beckmann_slopes(5, 1, w.mesh.ntris, 0.1)
    one, _, _ = orc.render(w.mesh, "R", w.endpoints, 24, 24, slopes=sl)
    three, _, _ = orc.render(w.mesh, "R", w.endpoints, 24, 24, slopes=np.repeat(sl, 3, axis=0))
    assert np.allclose(one, three, rtol=1e-14, atol=0)
    spec, _, _ = orc.render(w.mesh, "R", w.endpoints, 24, 24)
    zero, _, _ = orc.render(w.mesh, "R", w.endpoints, 24, 24, slopes=np.zeros((2, w.mesh.ntris, 2)))
    assert np.allclose(spec, zero, rtol=1e-14, atol=0)
    assert not np.allclose(one, spec)  # the offset moves the caustic


def test_image_files_roundtrip(tmp_path, orc):
    from paper_2405_13409_b200.image_io import read_pfm, write_pfm, write_ppm
    rad = np.random.default_rng(1).random((5, 7))
    write_pfm(str(tmp_path / "a.pfm"), rad)
    assert np.allclose(read_pfm(str(tmp_path / "a.pfm")), rad.astype(np.float32), rtol=0, atol=0)
    rgb = orc.tonemap_srgb(rad)
    write_ppm(str(tmp_path / "a.ppm"), rgb)
    b = open(tmp_path / "a.ppm", "rb").read()
    assert b.startswith(b"P6\n7 5\n255\n") and b[len(b"P6\n7 5\n255\n"):] == rgb.tobytes()
