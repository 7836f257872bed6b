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


def shoot(chain, tris, x0, xk1, u, v, eta_front=1.0, eta_back=1.0):
    """Forward exact shooting from x0 through (u,v) on T_1.  Returns (miss (...,3), u2, v2, ok).

    miss = (direction leaving the last vertex) - (unit direction to x_{k+1}).
    """
    T1 = tris[0]
    x1 = T1.X(u, v)
    n1 = _norm(T1.N(u, v))
    d0 = _norm(x1 - x0)
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


def brute_force(chain, mesh, tri_ids, x0, xk1, grid=512, eta_front=1.0, eta_back=1.0, margin=0.02):
    """All admissible chains for one (query, tuple): list of (u1, v1[, u2, v2])."""
    tris = [Tri(mesh, t) for t in np.atleast_1d(tri_ids)]
    x0 = np.asarray(x0, float)
    xk1 = np.asarray(xk1, float)
    s = np.linspace(-margin, 1 + margin, grid)
    U, V = np.meshgrid(s, s, indexing="ij")
    mask = U + V <= 1 + margin
    miss, _, _, ok = shoot(chain, tris, x0, xk1, U, V, eta_front, eta_back)
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
        u, v = U[i, j], V[i, j]
        m0, _, _, _ = shoot(chain, tris, x0, xk1, np.array(u), np.array(v), eta_front, eta_back)
        f1, f2 = _frame(_norm(m0 + 0))  # any fixed frame transverse works near the root
        target_dir = None
        # residual function G: miss projected on a frame perpendicular to the target direction
        def G(uv):
            m, u2, v2, okk = shoot(chain, tris, x0, xk1, np.array(uv[0]), np.array(uv[1]), eta_front, eta_back)
            return np.array([m[0], m[1], m[2]]), bool(okk), float(u2), float(v2)
        uv = np.array([u, v])
        g, okk, _, _ = G(uv)
        if not okk:
            continue
        for _ in range(60):
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
        if not okk or np.linalg.norm(g) > 1e-10:
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
