"""Pins of the oracle's two-bounce path, face-normal mode, contribution and flags (no GPU).

Every expected value comes from something other than the oracle's own formulas: image-source closed forms
for flat mirrors (SURVEY §8(c) fixed point 1 generalised to two mirrors), index-matched interfaces (free
space), the inverse-function-theorem Jacobian of the exact path-space solver in tests/bruteforce.py, the
camera-side and light-side brute-force sweeps (fixed point 4a/4b), and physical fold / edge / normal-incidence
constructions for the c14 flags.
"""
import numpy as np
import pytest

import bruteforce
from planted import planted_many
from paper_2405_13409_b200.workloads import Mesh

CHAINS2 = ["RR", "TT", "RT", "TR"]


def _solve1(orc, mesh, chain, x0, xk1, ids, **cfg):
    k = len(chain)
    return orc.solve(mesh, chain, np.array([[x0, xk1]]), offsets=np.array([0, 1], np.uint32),
                     tri_ids=np.array(ids, np.uint32), cfg=orc.default_config(cull=0, **cfg))


def _plane(P):
    g = np.cross(P[1] - P[0], P[2] - P[0])
    return P[0], g / np.linalg.norm(g)


def _mirror_point(x, P):
    p0, g = _plane(P)
    return x - 2 * np.dot(x - p0, g) * g


def _line_plane(a, b, P):
    p0, g = _plane(P)
    t = np.dot(p0 - a, g) / np.dot(b - a, g)
    return a + t * (b - a)


def _bary(x, P):
    M = np.stack([P[1] - P[0], P[2] - P[0]], 1)
    uv, *_ = np.linalg.lstsq(M, x - P[0], rcond=None)
    return uv


# ------------------------------------------------------------------ face mode (Table 2 "F")
def test_face_mode_flat_mirrors_rr_image_source(orc):
    """Two flat face-normal mirrors: the RR chain is the image-source construction (reflect x_3 across T_2's
    plane, that image across T_1's plane, straight line from x_0), and the point-light factor is J = L^2 with
    L the unfolded path length (a planar mirror maps the spherical wavefront onto a spherical one).  Reading
    R22 (constant n_2 in face mode) is what makes these systems solvable: under the interpolated structure
    kappa n_{2,0} is a factor common to a and b and det R(v) is rounding noise."""
    cases = planted_many(101, "RR", 40, face=True, size=0.15)
    assert len(cases) == 40
    for mesh, ids, x0, xk1, bary in cases:
        P1 = mesh.pos[mesh.tri[0]].astype(float)
        P2 = mesh.pos[mesh.tri[1]].astype(float)
        x3p = _mirror_point(xk1, P2)
        x3pp = _mirror_point(x3p, P1)
        x1 = _line_plane(x0, x3pp, P1)
        x2 = _line_plane(x1, x3p, P2)
        uv = np.concatenate([_bary(x1, P1), _bary(x2, P2)])
        L = np.linalg.norm(x3pp - x0)
        r = _solve1(orc, mesh, "RR", x0, xk1, ids)
        assert len(r.flagged_flags) == 0, r.flagged_flags
        assert r.n_solutions == 1
        # face normals are float32 roundings of the geometric normal: the shading plane is off by ~1e-7
        assert np.max(np.abs(r.bary[0] - uv)) < 1e-6
        assert abs((1.0 / r.contribution[0]) / (L * L) - 1) < 1e-6


@pytest.mark.parametrize("chain", ["RT", "TR", "TT"])
def test_face_mode_planted_recovered_unflagged(orc, chain):
    """Face-normal triangles on every vertex: 40/40 planted chains recovered unflagged, with the
    Eq. 3 residual < 1e-6 recomputed from scratch."""
    cases = planted_many(111, chain, 40, face=True, size=0.15)
    assert len(cases) == 40
    for mesh, ids, x0, xk1, bary in cases:
        r = _solve1(orc, mesh, chain, x0, xk1, ids)
        assert len(r.flagged_flags) == 0, (r.flagged_flags, bary)
        d = [np.max(np.abs(b - bary)) for b in r.bary]
        assert d and min(d) < 1e-6
        for b in r.bary:
            assert bruteforce.specular_residual(chain, mesh, ids, x0, xk1, b, mesh.eta_front, mesh.eta_back) < 1e-6


# ------------------------------------------------------------------ contribution (c15) closed forms, k = 2
def test_index_matched_interface_after_mirror_free_space(orc):
    """RT with eta = 1 on both sides of the interface: the refraction does not bend the ray, so the chain unfolds
    to the single-flat-mirror geometry: J = L^2, L = |x_1 - x_0| + |x_2 - x_1| + |x_3 - x_2| (SPEC S:551
    generalised to k = 2).  (An index-matched FIRST vertex is not used: its raw roots carry the sqrt
    surrogate's error, and Eq. 3's residual of a straight-through vertex is normalised by the floor of
    reading R3, so they miss the theta_admit gate -- a vacuous physical case.)"""
    chain = "RT"
    n = 0
    for mesh, ids, x0, xk1, bary in planted_many(121, chain, 12, size=0.15, eta=(1.0, 1.0), face=True):
        r = _solve1(orc, mesh, chain, x0, xk1, ids)
        for b, c in zip(r.bary, r.contribution):
            P1 = mesh.pos[mesh.tri[0]].astype(float)
            P2 = mesh.pos[mesh.tri[1]].astype(float)
            x1 = P1[0] + b[0] * (P1[1] - P1[0]) + b[1] * (P1[2] - P1[0])
            x2 = P2[0] + b[2] * (P2[1] - P2[0]) + b[3] * (P2[2] - P2[0])
            L = np.linalg.norm(x1 - x0) + np.linalg.norm(x2 - x1) + np.linalg.norm(xk1 - x2)
            assert abs((1.0 / c) / (L * L) - 1) < 1e-6
            n += 1
    assert n >= 8


@pytest.mark.parametrize("chain", ["R", "T"] + CHAINS2)
def test_contribution_matches_inverse_map_jacobian(orc, chain):
    """Curved (interpolated-normal) chains: the oracle's J (central differences of the LIGHT-side trace) equals
    1 / |det d(omega_light) / d(x_0 perp)| obtained by moving the camera and re-solving the chain with the
    polynomial-free exact-path Newton of tests/bruteforce.py (inverse function theorem).  No shared code, no
    shared method: one traces rays from the light, the other re-solves connections from perturbed cameras."""
    n = 0
    for mesh, ids, x0, xk1, bary in planted_many(131, chain, 10, size=0.15):
        r = _solve1(orc, mesh, chain, x0, xk1, ids)
        for b, c, f in zip(r.bary, r.contribution, r.flags):
            if f:
                continue
            Je = bruteforce.endpoint_jacobian(chain, mesh, ids, x0, xk1, b, mesh.eta_front, mesh.eta_back)
            assert abs((1.0 / c) / Je - 1) < 1e-6, (chain, 1.0 / c, Je)
            n += 1
    assert n >= 6


@pytest.mark.parametrize("chain", CHAINS2)
def test_two_bounce_scale_covariance(orc, chain):
    """Doubling the scene scale quarters the contribution, two bounces."""
    n = 0
    for mesh, ids, x0, xk1, bary in planted_many(141, chain, 5, size=0.15):
        r1 = _solve1(orc, mesh, chain, x0, xk1, ids)
        m2 = Mesh(mesh.pos * 2, mesh.nrm, mesh.tri, mesh.eta_front, mesh.eta_back)
        r2 = _solve1(orc, m2, chain, 2 * x0, 2 * xk1, ids)
        assert r2.n_solutions == r1.n_solutions
        assert np.allclose(r2.bary, r1.bary, atol=1e-8)
        assert np.allclose(r2.contribution * 4, r1.contribution, rtol=1e-6)
        n += r1.n_solutions
    assert n >= 3


# ------------------------------------------------------------------ completeness: brute force (4a) + light side (4b)
def _batch(chain, n, seed):
    """n planted configurations merged into one mesh; tuple list = the planted pair + 2 decoy pairs per query."""
    cases = planted_many(seed, chain, n, size=0.15)
    pos, nrm, tri, eps = [], [], [], []
    for i, (m, ids, x0, xk1, bary) in enumerate(cases):
        pos.append(m.pos)
        nrm.append(m.nrm)
        tri.append(m.tri + 6 * i)
        eps.append([x0, xk1])
    mesh = Mesh(np.concatenate(pos), np.concatenate(nrm), np.concatenate(tri).astype(np.uint32),
                cases[0][0].eta_front, cases[0][0].eta_back)
    rng = np.random.default_rng(seed + 1)
    offsets, ids = [0], []
    for i in range(len(cases)):
        tl = [(2 * i, 2 * i + 1)]
        while len(tl) < 3:  # two distinct decoy pairs
            j, l = rng.integers(0, len(cases), 2)
            if (2 * int(j), 2 * int(l) + 1) not in tl:
                tl.append((2 * int(j), 2 * int(l) + 1))
        for a, b in tl:
            ids += [a, b]
        offsets.append(offsets[-1] + len(tl))
    return mesh, np.array(eps, float), np.array(offsets, np.uint32), np.array(ids, np.uint32)


@pytest.mark.parametrize("chain", CHAINS2)
def test_two_bounce_bruteforce_completeness(orc, chain):
    """<= 64 tuples per chain: every oracle chain is confirmed by the light-side shot (the exact ray from
    x_3 back through the chain passes within 1e-9 of x_0) and found by both brute-force sweeps; every chain
    either sweep finds is in the oracle's set unless its tuple is flagged, or it is one of the documented
    100-piece scan misses, whose rate is bounded (SPEC S:714 recall >= 0.95)."""
    mesh, ep, off, ids = _batch(chain, 12, 151)
    r = orc.solve(mesh, chain, ep, offsets=off, tri_ids=ids)
    assert r.report["pairs_in"] <= 64
    flagged = {(int(q), int(a), int(b)) for q, (a, b) in zip(r.flagged_query, r.flagged_tuple)}
    n_bf = n_miss = n_orc = 0
    for qi in range(len(ep)):
        x0, xk1 = ep[qi]
        for t in range(off[qi], off[qi + 1]):
            tup = [int(ids[2 * t]), int(ids[2 * t + 1])]
            mine = [r.bary[i] for i in range(r.n_solutions) if r.query[i] == qi and list(r.tuple[i]) == tup]
            cam = bruteforce.brute_force(chain, mesh, tup, x0, xk1, grid=384, eta_front=mesh.eta_front,
                                         eta_back=mesh.eta_back)
            lit = bruteforce.brute_force_light(chain, mesh, tup, x0, xk1, grid=384, eta_front=mesh.eta_front,
                                               eta_back=mesh.eta_back)
            for b in mine:  # confirmation (4b) + presence in both sweeps
                n_orc += 1
                assert bruteforce.light_shot_miss(chain, mesh, tup, x0, xk1, b, mesh.eta_front,
                                                  mesh.eta_back) < 1e-9
                assert any(np.max(np.abs(b - np.array(c))) < 1e-6 for c in cam), (qi, tup, b, cam)
                assert any(np.max(np.abs(b - np.array(c))) < 1e-6 for c in lit), (qi, tup, b, lit)
            if (qi, *tup) in flagged:
                continue
            for c in set(cam) | set(lit):
                n_bf += 1
                if not any(np.max(np.abs(np.array(c) - b)) < 1e-6 for b in mine):
                    n_miss += 1
    assert n_orc >= 10
    assert n_miss <= 0.05 * max(n_bf, 1), (n_miss, n_bf)


def test_one_bounce_light_side_confirms_c1(orc):
    """C1 patch: every oracle chain is confirmed by the light-side shot and found by the light-side sweep; the
    light-side sweep finds nothing the oracle missed outside flagged tuples (fixed point 4b, k = 1)."""
    from paper_2405_13409_b200.workloads import patch_c1
    w = patch_c1()
    r = orc.solve(w.mesh, "R", w.endpoints, cfg=orc.default_config(cull=0))
    x0, xk1 = w.endpoints[0]
    flagged = set(map(int, r.flagged_tuple[:, 0])) if len(r.flagged_flags) else set()
    n = 0
    for t in range(w.mesh.ntris):
        mine = [r.bary[i] for i in range(r.n_solutions) if r.tuple[i, 0] == t]
        for b in mine:
            assert bruteforce.light_shot_miss("R", w.mesh, [t], x0, xk1, b) < 1e-9
        if t in flagged:
            continue
        lit = bruteforce.brute_force_light("R", w.mesh, [t], x0, xk1, grid=96)
        assert len(lit) == len(mine), (t, mine, lit)
        for c in lit:
            assert any(np.max(np.abs(np.array(c) - b)) < 1e-6 for b in mine)
        n += len(mine)
    assert n >= 1


# ------------------------------------------------------------------ c14 flags fire where they must, and only there
def _concave_mirror(kappa=0.8):
    P = np.array([[-1, -1, 0], [1.2, -0.9, 0], [-0.8, 1.1, 0]], float)
    c = P.mean(0)
    N = np.array([np.array([0, 0, 1.0]) - kappa * (p - c) for p in P])
    N /= np.linalg.norm(N, axis=1)[:, None]
    return Mesh(P.astype(np.float32), N.astype(np.float32), np.array([[0, 1, 2]], np.uint32))


def test_near_tangent_flag_at_folds(orc):
    """Folds (caustics) of a focusing interpolated-normal mirror: two chains merge into a double root of r(v).
    Walking the light towards a fold, the tuple must be flagged NEAR_TANGENT on both sides of the transition
    (bisected to 1e-15 in the walk parameter), and unflagged half way back to the start, where the two chains
    are well separated."""
    mesh = _concave_mirror()
    rng = np.random.default_rng(0)
    Q = 4000
    ep = np.zeros((Q, 2, 3))
    ep[:, 0] = rng.uniform(-2, 2, (Q, 3)) * [1, 1, 0] + [0, 0, 1] * rng.uniform(0.2, 3, (Q, 1))
    ep[:, 1] = rng.uniform(-2, 2, (Q, 3)) * [1, 1, 0] + [0, 0, 1] * rng.uniform(0.2, 3, (Q, 1))
    cfg = orc.default_config(cull=0)
    r = orc.solve(mesh, "R", ep, cfg=cfg)
    two = np.where(np.bincount(r.query, minlength=Q) == 2)[0]

    def at(x0, x2):
        rr = orc.solve(mesh, "R", np.array([[x0, x2]]), cfg=cfg)
        return rr, (int(rr.flagged_flags[0]) if len(rr.flagged_flags) else 0)

    folds = 0
    for q in two:
        x0, x2 = ep[q]
        for trial in range(6):
            d = rng.normal(size=3)
            d /= np.linalg.norm(d)
            lo, hi = 0.0, None
            for s in np.linspace(0, 1, 101)[1:]:
                if at(x0, x2 + s * d)[0].n_solutions != 2:
                    hi = s
                    break
                lo = s
            if hi is None or at(x0, x2 + hi * d)[0].n_solutions == 1 and at(x0, x2 + hi * d)[1] == 0:
                continue
            for _ in range(60):
                m = 0.5 * (lo + hi)
                if at(x0, x2 + m * d)[0].n_solutions == 2:
                    lo = m
                else:
                    hi = m
            ra, fa = at(x0, x2 + lo * d)
            if np.max(np.abs(ra.bary[0] - ra.bary[1])) > 1e-3:
                continue  # a chain left through an edge: not a fold
            rb, fb = at(x0, x2 + hi * d)
            assert fa & orc.FLAG_NEAR_TANGENT and fb & orc.FLAG_NEAR_TANGENT, (fa, fb)
            rm, fm = at(x0, x2 + 0.5 * lo * d)
            if rm.n_solutions == 2 and np.max(np.abs(rm.bary[0] - rm.bary[1])) > 1e-2:
                assert fm == 0, fm
            folds += 1
            break
    assert folds >= 3


def test_boundary_flag_on_edge_chain(orc):
    """A planted chain whose vertex lies exactly on the edge u + v = 1 is flagged BOUNDARY; the same geometry with
    the vertex 1e-3 inside is not.  (The u + v = 1 edge is the one both labelings of reading R1 share; on the
    solver's v = 0 / v = 1 edges a root just outside [0, 1] is not isolated at all (the paper's interval,
    PAPER.md:608), so no candidate exists there to flag -- DESIGN.md reading R11.)"""
    from planted import _n, _reflect
    rng = np.random.default_rng(3)
    n_edge = 0
    for trial in range(40):
        P = rng.normal(size=(3, 3)) * [1, 1, 0.1]
        P = P.astype(np.float32).astype(np.float64)
        g = np.cross(P[1] - P[0], P[2] - P[0])
        if g[2] < 0:
            P = P[[0, 2, 1]]
            g = -g
        if np.linalg.norm(g) < 0.3:
            continue
        N = np.array([_n(g / np.linalg.norm(g) + 0.2 * rng.normal(size=3)) for _ in range(3)])
        N = N.astype(np.float32).astype(np.float64)
        mesh = Mesh(P.astype(np.float32), N.astype(np.float32), np.array([[0, 1, 2]], np.uint32))
        for v1, expect in ((0.6, True), (0.6 - 1e-3, False)):
            u1 = 0.4
            x1 = P[0] + u1 * (P[1] - P[0]) + v1 * (P[2] - P[0])
            n1 = _n(N[0] + u1 * (N[1] - N[0]) + v1 * (N[2] - N[0]))
            w = _n(n1 + 0.5 * rng.normal(size=3))
            if np.dot(w, n1) < 0.3 or np.dot(w, g) < 0.3:
                break
            x0 = x1 + 1.5 * w
            w1 = _reflect(_n(x1 - x0), n1)
            if np.dot(w1, n1) < 0.2 or np.dot(w1, g) < 0.2:
                break
            x2 = x1 + 1.2 * w1
            r = orc.solve(mesh, "R", np.array([[x0, x2]]), cfg=orc.default_config(cull=0))
            f = int(r.flagged_flags[0]) if len(r.flagged_flags) else 0
            assert bool(f & orc.FLAG_BOUNDARY) == expect, (v1, f, r.bary)
            n_edge += expect
    assert n_edge >= 10


def test_degenerate_flag_at_normal_incidence(orc):
    """x_0 and x_2 on the normal line through the centroid: the incidence plane is undefined (reading R1 l_c = 0),
    the tuple is flagged DEGENERATE; a small lateral offset removes the flag."""
    mesh = _concave_mirror(0.0)
    c = mesh.pos.astype(float).mean(0)
    n = mesh.nrm[0].astype(float)
    r = orc.solve(mesh, "R", np.array([[c + 1.0 * n, c + 2.0 * n]]), cfg=orc.default_config(cull=0))
    assert len(r.flagged_flags) == 1 and r.flagged_flags[0] & orc.FLAG_DEGENERATE
    r = orc.solve(mesh, "R", np.array([[c + 1.0 * n + [0.3, 0, 0], c + 2.0 * n]]), cfg=orc.default_config(cull=0))
    assert len(r.flagged_flags) == 0 and r.n_solutions == 1


def test_generic_planted_chains_unflagged(orc):
    """Generic planted chains (interior, transversal, away from folds) carry no flag: the flags are rare where
    nothing is special (the parity harness bounds the flagged fraction at 2%)."""
    tot = fl = 0
    for chain in ("R", "T") + tuple(CHAINS2):
        for mesh, ids, x0, xk1, bary in planted_many(161, chain, 20, size=0.15):
            r = _solve1(orc, mesh, chain, x0, xk1, ids)
            tot += 1
            fl += len(r.flagged_flags) > 0
    assert fl <= 0.02 * tot, (fl, tot)


# ------------------------------------------------------------------ visibility
def _seg_tri_numpy(a, b, P):
    """Independent segment/triangle test: intersect the segment with the triangle's plane, then the barycentric
    coordinates of the hit from signed sub-triangle areas (not Moller-Trumbore).  Returns (hit, t)."""
    n = np.cross(P[1] - P[0], P[2] - P[0])
    da, db = np.dot(a - P[0], n), np.dot(b - P[0], n)
    if da * db > 0 or da == db:
        return False, None
    t = da / (da - db)
    x = a + t * (b - a)
    A = [np.dot(np.cross(P[(i + 1) % 3] - x, P[(i + 2) % 3] - x), n) for i in range(3)]
    return all(s >= 0 for s in A) or all(s <= 0 for s in A), t


def test_visibility_blocker_closed_form(orc):
    """A flat mirror chain (S:520 geometry) with a small blocker triangle straddling the segment x_0 -> x_1: the chain
    is rejected with visibility on, kept with visibility off or with the blocker moved aside; a blocker across
    x_1 -> x_2 rejects it too; the mirror triangle itself never blocks its own vertex."""
    pos = np.array([[-1, -1, 0], [2, -1, 0], [-1, 2, 0]], np.float32)
    nrm = np.tile([0, 0, 1], (3, 1)).astype(np.float32)
    mesh = Mesh(pos, nrm, np.array([[0, 1, 2]], np.uint32))
    ep = np.array([[[0, 0, 1], [1, 0, 1]]], float)
    x1 = np.array([0.5, 0, 0])

    def blocker(center):
        c = np.asarray(center, float)
        P = np.array([c + [-0.1, -0.1, 0.02], c + [0.1, -0.1, -0.02], c + [0.0, 0.15, 0.0]], np.float32)
        return Mesh(P, np.tile([0, 0, 1], (3, 1)).astype(np.float32), np.array([[0, 1, 2]], np.uint32))
    on = orc.default_config(cull=0, visibility=1)
    r = orc.solve(mesh, "R", ep, cfg=orc.default_config(cull=0), occluders=blocker(0.5 * (ep[0, 0] + x1)))
    assert r.n_solutions == 1
    r = orc.solve(mesh, "R", ep, cfg=on, occluders=blocker(0.5 * (ep[0, 0] + x1)))
    assert r.n_solutions == 0 and r.report["rej_visibility"] == 1 and r.per_query[0] == 0
    r = orc.solve(mesh, "R", ep, cfg=on, occluders=blocker(0.5 * (ep[0, 1] + x1)))
    assert r.n_solutions == 0 and r.report["rej_visibility"] == 1
    r = orc.solve(mesh, "R", ep, cfg=on, occluders=blocker(0.5 * (ep[0, 0] + x1) + [0, 0.6, 0]))
    assert r.n_solutions == 1 and r.report["rej_visibility"] == 0
    r = orc.solve(mesh, "R", ep, cfg=on)
    assert r.n_solutions == 1


@pytest.mark.parametrize("chain", ["R", "RR", "TT"])
def test_visibility_matches_independent_segment_test(orc, chain):
    """Random occluders over planted chains: with visibility on, the oracle returns exactly the chains whose every
    segment misses every scene triangle (other than the chain's own triangles at the segment's ends) according to
    an independent numpy segment test (plane crossing + signed areas)."""
    rng = np.random.default_rng(181)
    cases = planted_many(191, chain, 30, size=0.15)
    n_blocked = n_kept = 0
    for mesh, ids, x0, xk1, bary in cases:
        # occluders: small random triangles near the chain's segments
        r0 = _solve1(orc, mesh, chain, x0, xk1, ids)
        if r0.n_solutions == 0:
            continue
        b = r0.bary[0]
        tris = [mesh.pos[mesh.tri[t]].astype(float) for t in ids]
        xs = [x0] + [tris[i][0] + b[2 * i] * (tris[i][1] - tris[i][0]) + b[2 * i + 1] * (tris[i][2] - tris[i][0])
                     for i in range(len(ids))] + [xk1]
        occ = []
        for _ in range(6):
            i = rng.integers(0, len(xs) - 1)
            c = xs[i] + rng.uniform(0.2, 0.8) * (xs[i + 1] - xs[i]) + rng.normal(size=3) * 0.08
            occ.append(c + rng.normal(size=(3, 3)) * 0.06)
        opos = np.concatenate(occ).astype(np.float32)
        omesh = Mesh(opos, np.tile([0, 0, 1], (len(opos), 1)).astype(np.float32),
                     np.arange(len(opos), dtype=np.uint32).reshape(-1, 3))
        r1 = orc.solve(mesh, chain, np.array([[x0, xk1]]), offsets=np.array([0, 1], np.uint32),
                       tri_ids=np.array(ids, np.uint32), cfg=orc.default_config(cull=0, visibility=1), occluders=omesh)
        kept = {tuple(np.round(x, 12)) for x in r1.bary}
        for bb in r0.bary:
            pts = [x0] + [tris[i][0] + bb[2 * i] * (tris[i][1] - tris[i][0]) + bb[2 * i + 1] * (tris[i][2] - tris[i][0])
                          for i in range(len(ids))] + [xk1]
            blocked = False
            for s in range(len(pts) - 1):
                for P in [opos[3 * j:3 * j + 3].astype(float) for j in range(len(occ))]:
                    hit, t = _seg_tri_numpy(pts[s], pts[s + 1], P)
                    if hit and 1e-6 < t < 1 - 1e-6:
                        blocked = True
            assert blocked == (tuple(np.round(bb, 12)) not in kept), (chain, bb, blocked)
            n_blocked += blocked
            n_kept += not blocked
    assert n_blocked >= 3 and n_kept >= 3, (n_blocked, n_kept)
