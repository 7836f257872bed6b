"""Independent brute-force specular-chain finder (tests only).

Shares nothing with oracle/ or the CUDA path: it never builds a polynomial.  It sweeps a dense
barycentric grid over T_1 in EXACT path space (true normalisation, true sqrt in Snell's law),
takes local minima of the shooting residual, polishes them with damped Newton and keeps
converged, in-domain, side-consistent chains (SURVEY §8(c) fixed point 4a).  For k=1 the
sweep is over x_1; for k=2 it shoots from x_0 through x_1 on T_1, intersects T_2's plane, and
measures the miss against x_3.
"""
from __future__ import annotations

import numpy as np


def _norm(v):
    return v / np.linalg.norm(v, axis=-1, keepdims=True)


def _reflect(d, n):
    return d - 2 * np.sum(d * n, -1, keepdims=True) * n


def _refract(d, n, eta_in, eta_out):
    ep = eta_in / eta_out
    ci = -np.sum(d * n, -1, keepdims=True)
    n = np.where(ci < 0, -n, n)
    ci = np.abs(ci)
    k = 1 - ep * ep * (1 - ci * ci)
    ok = (k >= 0)[..., 0]
    t = ep * d + (ep * ci - np.sqrt(np.maximum(k, 0))) * n
    return t, ok


class Tri:
    def __init__(self, mesh, t):
        vi = mesh.tri[int(t)]
        self.p = mesh.pos[vi].astype(np.float64)
        self.n = mesh.nrm[vi].astype(np.float64)
        self.e1 = self.p[1] - self.p[0]
        self.e2 = self.p[2] - self.p[0]
        self.g = np.cross(self.e1, self.e2)

    def X(self, u, v):
        return self.p[0] + u[..., None] * self.e1 + v[..., None] * self.e2

    def N(self, u, v):
        return self.n[0] + u[..., None] * (self.n[1] - self.n[0]) + v[..., None] * (self.n[2] - self.n[0])

    def hit(self, o, d):
        P = np.cross(d, self.e2)
        det = np.sum(P * self.e1, -1)
        s = o - self.p[0]
        u = np.sum(s * P, -1) / det
        Q = np.cross(s, self.e1)
        v = np.sum(d * Q, -1) / det
        t = np.sum(self.e2 * Q, -1) / det
        return u, v, t


def _side_eta(x, tri, eta_front, eta_back):
    return np.where(np.sum((x - tri.p[0]) * tri.g, -1) > 0, eta_front, eta_back)


def shoot(chain, tris, x0, xk1, u, v, eta_front=1.0, eta_back=1.0, media=None):
    """Forward exact shooting from x0 through (u,v) on T_1.  Returns (miss (...,3), u2, v2, ok).

    miss = (direction leaving the last vertex) - (unit direction to x_{k+1}).  media: explicit (eta_0, eta_1,
    eta_2) along the chain (the light-side sweep passes the forward chain's media reversed); default: eta_0 from
    x0's side of T_1, flipped at every refraction, and for k = 2 the far side of T_2 from x1's side.
    """
    T1 = tris[0]
    x1 = T1.X(u, v)
    n1 = _norm(T1.N(u, v))
    d0 = _norm(x1 - x0)
    if media is not None:
        eta0, eta1 = media[0], media[1]
    else:
        eta0 = _side_eta(np.asarray(x0)[None], T1, eta_front, eta_back)[0]
        eta1 = eta0 if chain[0] == "R" else (eta_back if eta0 == eta_front else eta_front)
    ok = np.ones(u.shape, bool)
    if chain[0] == "R":
        w1 = _reflect(d0, n1)
    else:
        w1, ok1 = _refract(d0, n1, eta0, eta1)
        ok &= ok1
    if len(chain) == 1:
        return w1 - _norm(xk1 - x1), u * 0, v * 0, ok
    T2 = tris[1]
    w1 = _norm(w1)
    u2, v2, t = T2.hit(x1, w1)
    ok &= t > 0
    x2 = x1 + t[..., None] * w1
    n2 = _norm(T2.N(u2, v2))
    eta2s = _side_eta(x1, T2, eta_front, eta_back)  # medium x1 is in w.r.t. T2
    eta_far = np.where(eta2s == eta_front, eta_back, eta_front)
    if media is not None:
        eta_far = media[2] * np.ones_like(eta_far)
    if chain[1] == "R":
        w2 = _reflect(w1, n2)
    else:
        w2, ok2 = _refract(w1, n2, eta1 * np.ones_like(eta_far)[..., None], eta_far[..., None])
        ok &= ok2
        ok &= eta2s == eta1
    return _norm(w2) - _norm(xk1 - x2), u2, v2, ok


def _frame(w):
    a = np.array([1.0, 0, 0]) if abs(w[0]) < 0.6 else np.array([0, 1.0, 0])
    f1 = _norm(np.cross(w, a))
    return f1, np.cross(w, f1)


def brute_force(chain, mesh, tri_ids, x0, xk1, grid=512, eta_front=1.0, eta_back=1.0, margin=0.02, media=None):
    """All admissible chains for one (query, tuple): list of (u1, v1[, u2, v2])."""
    tris = [Tri(mesh, t) for t in np.atleast_1d(tri_ids)]
    x0 = np.asarray(x0, float)
    xk1 = np.asarray(xk1, float)
    s = np.linspace(-margin, 1 + margin, grid)
    U, V = np.meshgrid(s, s, indexing="ij")
    mask = U + V <= 1 + margin
    miss, _, _, ok = shoot(chain, tris, x0, xk1, U, V, eta_front, eta_back, media)
    F = np.linalg.norm(miss, axis=-1)
    F = np.where(ok & mask, F, np.inf)
    # local minima on the grid (8-neighbourhood)
    Fp = np.pad(F, 1, constant_values=np.inf)
    is_min = np.ones_like(F, bool)
    for di in (-1, 0, 1):
        for dj in (-1, 0, 1):
            if di == 0 and dj == 0:
                continue
            is_min &= F <= Fp[1 + di:1 + di + grid, 1 + dj:1 + dj + grid]
    seeds = np.argwhere(is_min & (F < 0.05))
    sols = []
    for i, j in seeds:
        uv, gn, u2, v2, okk = _newton(chain, tris, x0, xk1, np.array([U[i, j], V[i, j]]), eta_front, eta_back,
                                      media=media)
        if not okk or gn > 1e-10:
            continue
        u, v = uv
        inside = u >= -1e-9 and v >= -1e-9 and u + v <= 1 + 1e-9
        if len(tris) == 2:
            inside = inside and u2 >= -1e-9 and v2 >= -1e-9 and u2 + v2 <= 1 + 1e-9
        if not inside:
            continue
        if not _sides_ok(chain, tris, x0, xk1, u, v, u2, v2):
            continue
        cand = (u, v) if len(tris) == 1 else (u, v, u2, v2)
        if all(np.max(np.abs(np.array(cand) - np.array(c))) > 1e-7 for c in sols):
            sols.append(cand)
    return sorted(sols)


def _newton(chain, tris, x0, xk1, uv, eta_front, eta_back, iters=60, media=None):
    """Damped Gauss-Newton on the exact shooting miss (3 components) from the seed uv on T_1.  Returns
    (uv, |miss|, u2, v2, ok)."""
    def G(p):
        m, u2, v2, okk = shoot(chain, tris, x0, xk1, np.array(p[0]), np.array(p[1]), eta_front, eta_back, media)
        return np.array([m[0], m[1], m[2]]), bool(okk), float(u2), float(v2)
    uv = np.asarray(uv, float)
    g, okk, _, _ = G(uv)
    if not okk:
        return uv, np.inf, 0.0, 0.0, False
    for _ in range(iters):
        h = 1e-7
        J = np.zeros((3, 2))
        for c in range(2):
            e = np.zeros(2)
            e[c] = h
            gp, _, _, _ = G(uv + e)
            gm, _, _, _ = G(uv - e)
            J[:, c] = (gp - gm) / (2 * h)
        step, *_ = np.linalg.lstsq(J, -g, rcond=None)
        lam = 1.0
        gn = None
        while lam > 1e-4:
            gn, okn, _, _ = G(uv + lam * step)
            if okn and np.linalg.norm(gn) < np.linalg.norm(g):
                break
            lam *= 0.5
        if gn is None or lam <= 1e-4:
            break
        uv = uv + lam * step
        g = gn
        if np.linalg.norm(g) < 1e-14:
            break
    g, okk, u2, v2 = G(uv)
    return uv, float(np.linalg.norm(g)), u2, v2, okk


def _sides_ok(chain, tris, x0, xk1, u, v, u2, v2):
    pts = [np.asarray(x0, float)]
    ns = []
    for i, t in enumerate(tris):
        uu, vv = (u, v) if i == 0 else (u2, v2)
        pts.append(t.X(np.array(uu), np.array(vv)))
        ns.append(_norm(t.N(np.array(uu), np.array(vv))))
    pts.append(np.asarray(xk1, float))
    for i, t in enumerate(tris):
        xp, x, xn = pts[i], pts[i + 1], pts[i + 2]
        spn, snn = np.dot(xp - x, ns[i]), np.dot(xn - x, ns[i])
        spg, sng = np.dot(xp - x, t.g), np.dot(xn - x, t.g)
        if not spn * spg > 0:
            return False
        if chain[i] == "R" and not (spn * snn > 0 and spg * sng > 0):
            return False
        if chain[i] == "T" and not (spn * snn < 0 and spg * sng < 0):
            return False
    return True


def specular_residual(chain, mesh, tri_ids, x0, xk1, bary, eta_front=1.0, eta_back=1.0):
    """max_i |h^_i x n^_i| (Eq. 3) recomputed from scratch for a returned chain."""
    tris = [Tri(mesh, t) for t in np.atleast_1d(tri_ids)]
    pts = [np.asarray(x0, float)]
    ns = []
    for i, t in enumerate(tris):
        u, v = np.array(bary[2 * i]), np.array(bary[2 * i + 1])
        pts.append(t.X(u, v))
        ns.append(_norm(t.N(u, v)))
    pts.append(np.asarray(xk1, float))
    eta = [_side_eta(pts[0][None], tris[0], eta_front, eta_back)[0]]
    for i, t in enumerate(tris):
        if chain[i] == "R":
            eta.append(eta[-1])
        else:
            eta.append(eta_back if eta[-1] == eta_front else eta_front)
    worst = 0.0
    for i in range(len(tris)):
        dp = _norm(pts[i + 1] - pts[i])
        dn = _norm(pts[i + 2] - pts[i + 1])
        h = eta[i + 1] * dn - eta[i] * dp
        worst = max(worst, np.linalg.norm(np.cross(_norm(h), ns[i])))
    return worst


# ---------------------------------------------------------------- light-side ray shooting
def brute_force_light(chain, mesh, tri_ids, x0, xk1, grid=512, eta_front=1.0, eta_back=1.0, margin=0.02):
    """The same exact-path-space sweep run from the LIGHT: a grid over T_k's barycentrics, rays shot from
    x_{k+1} through x_k back along the reversed chain, the miss measured against x_0.  Returns the chains in
    the forward labeling (u1, v1[, u2, v2]), sorted.  It is a different parametrisation of the solution set
    (other triangle, other shooting origin), so it confirms and completes the camera-side sweep."""
    ids = list(np.atleast_1d(tri_ids))[::-1]
    fwd = _media(chain, [Tri(mesh, t) for t in np.atleast_1d(tri_ids)], x0, eta_front, eta_back)
    if len(chain) == 2 and chain[1] == "T":
        # forward rule of the camera sweep: the medium beyond T_2 is the far side of T_2 from x_1
        fwd[2] = None
    rev = brute_force(chain[::-1], mesh, ids, xk1, x0, grid=grid, eta_front=eta_front, eta_back=eta_back,
                      margin=margin, media=None if None in fwd else fwd[::-1])
    out = []
    for s in rev:
        s = np.asarray(s)
        out.append(tuple(s.reshape(-1, 2)[::-1].ravel()))
    return sorted(out)


def light_shot_miss(chain, mesh, tri_ids, x0, xk1, bary, eta_front=1.0, eta_back=1.0):
    """Distance from x_0 of the ray shot from the light x_{k+1} through the chain's last vertex and scattered
    exactly (true normalisation, true sqrt) back through every vertex: ~0 for a genuine chain."""
    tris = [Tri(mesh, t) for t in np.atleast_1d(tri_ids)]
    k = len(tris)
    b = np.asarray(bary, float).reshape(-1, 2)
    xk = tris[-1].X(np.array(b[-1, 0]), np.array(b[-1, 1]))
    eta = _media(chain, tris, x0, eta_front, eta_back)
    o, d = np.asarray(xk1, float), _norm(xk - np.asarray(xk1, float))
    for i in range(k - 1, -1, -1):
        u, v, t = tris[i].hit(o, d)
        if not t > 0:
            return np.inf
        x = o + t * d
        n = _norm(tris[i].N(np.array(u), np.array(v)))
        if chain[i] == "R":
            d = _norm(_reflect(d, n))
        else:
            d2, ok = _refract(d, n, eta[i + 1], eta[i])
            if not ok:
                return np.inf
            d = _norm(d2)
        o = x
    w = np.asarray(x0, float) - o
    return float(np.linalg.norm(w - np.dot(w, d) * d)) if np.dot(w, d) > 0 else np.inf


def _media(chain, tris, x0, eta_front, eta_back):
    """eta_0 .. eta_k along the chain (x_0's side of T_1, flipped at every refraction)."""
    eta = [float(_side_eta(np.asarray(x0, float)[None], tris[0], eta_front, eta_back)[0])]
    for c in chain:
        eta.append(eta[-1] if c == "R" else (eta_back if eta[-1] == eta_front else eta_front))
    return eta


def endpoint_jacobian(chain, mesh, tri_ids, x0, xk1, bary, eta_front=1.0, eta_back=1.0, h=1e-6):
    """The contribution's J (c15, reading R12: |det d(position on the plane through x_0 perpendicular to d_0) /
    d(emission direction at the light x_{k+1})|) computed the other way round, by the inverse function theorem:
    move the CAMERA x_0 by +-h along the two frame axes of that plane, re-solve the chain there (exact-path
    Newton from the known solution, no polynomials), read the emission direction omega = (x_k - x_{k+1})^ of
    the re-solved chain, and J = 1 / |det d(omega) / d(x_0 perp)| (central differences + Richardson).  It never
    traces from the light, so it pins the oracle's light-side finite differences independently."""
    tris = [Tri(mesh, t) for t in np.atleast_1d(tri_ids)]
    k = len(tris)
    b = np.asarray(bary, float).reshape(-1, 2)
    x0 = np.asarray(x0, float)
    xk1 = np.asarray(xk1, float)
    x1 = tris[0].X(np.array(b[0, 0]), np.array(b[0, 1]))
    xk = tris[-1].X(np.array(b[-1, 0]), np.array(b[-1, 1]))
    dref = _norm(x0 - x1)
    c1, c2 = _frame(dref)
    w = _norm(xk - xk1)
    b1, b2 = _frame(w)

    def omega(x0p):
        uv, gn, u2, v2, ok = _newton(chain, tris, x0p, xk1, b[0], eta_front, eta_back)
        assert ok and gn < 1e-13, (gn, ok)
        xl = tris[0].X(np.array(uv[0]), np.array(uv[1])) if k == 1 else tris[1].X(np.array(u2), np.array(v2))
        om = _norm(xl - xk1)
        return np.array([np.dot(om, b1), np.dot(om, b2)])

    def deriv(e, hh):
        return (omega(x0 + hh * e) - omega(x0 - hh * e)) / (2 * hh)
    j1 = (4 * deriv(c1, h / 2) - deriv(c1, h)) / 3
    j2 = (4 * deriv(c2, h / 2) - deriv(c2, h)) / 3
    return 1.0 / abs(j1[0] * j2[1] - j1[1] * j2[0])
