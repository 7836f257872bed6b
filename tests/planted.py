"""Planted specular chains built by FORWARD tracing (tests only; no polynomial arithmetic).

Pick x_1 on T_1, a camera point x_0, scatter the ray exactly (mirror law / Snell's law with the
normalised interpolated normal, Eq. 3), build T_2 around the hit point for k=2, scatter
again and put the light x_{k+1} on the outgoing ray.  The planted barycentrics are then a known
solution of the specular constraints.
"""
from __future__ import annotations

import numpy as np

from paper_2405_13409_b200.workloads import Mesh


def _n(v):
    return v / np.linalg.norm(v)


def _reflect(d, n):
    return d - 2 * np.dot(d, n) * n


def _refract(d, n, e_in, e_out):
    ep = e_in / e_out
    ci = -np.dot(d, n)
    if ci < 0:
        n = -n
        ci = -ci
    k = 1 - ep * ep * (1 - ci * ci)
    if k < 0:
        return None
    return ep * d + (ep * ci - np.sqrt(k)) * n


def _tri_around(rng, x, normal, size, tilt, face=False):
    """Random triangle containing x (barycentrics returned) with geometric normal ~ `normal`."""
    a = _n(np.cross(normal, rng.normal(size=3)))
    b = np.cross(normal, a)
    while True:
        ang = np.sort(rng.uniform(0, 2 * np.pi, 3))
        if np.max(np.diff(np.concatenate([ang, [ang[0] + 2 * np.pi]]))) < np.pi * 0.9:
            break
    r = size * rng.uniform(0.6, 1.4, 3)
    P = np.array([x + r[i] * (np.cos(ang[i]) * a + np.sin(ang[i]) * b) for i in range(3)])
    P = P.astype(np.float32).astype(np.float64)
    g = np.cross(P[1] - P[0], P[2] - P[0])
    if np.dot(g, normal) < 0:
        P = P[[0, 2, 1]]
        g = -g
    gh = _n(g)
    if face:
        N = np.tile(gh, (3, 1))
    else:
        N = np.array([_n(gh + tilt * rng.normal(size=3)) for _ in range(3)])
    N = N.astype(np.float32).astype(np.float64)
    # barycentrics of the projection of x onto the plane
    e1, e2 = P[1] - P[0], P[2] - P[0]
    M = np.stack([e1, e2], 1)
    uv, *_ = np.linalg.lstsq(M, x - P[0], rcond=None)
    return P, N, uv


def planted(rng, chain: str, size=0.2, tilt=0.2, face=False, dist=(1.0, 3.0), eta=(1.0, 1.5)):
    """Returns (mesh, tri_ids, x0, xk1, bary_planted) or None if the construction failed."""
    eta_front, eta_back = eta
    # T_1 facing +z; x_1 at its interior point
    c = rng.uniform(-0.5, 0.5, 3) * np.array([1, 1, 0.1])
    P1, N1, uv1 = _tri_around(rng, c, _n(np.array([0, 0, 1.0]) + 0.3 * rng.normal(size=3)), size, tilt, face)
    u1, v1 = rng.uniform(0.05, 0.9), 0.0
    v1 = rng.uniform(0.05, 0.95 - u1)
    x1 = P1[0] + u1 * (P1[1] - P1[0]) + v1 * (P1[2] - P1[0])
    n1 = _n(N1[0] + u1 * (N1[1] - N1[0]) + v1 * (N1[2] - N1[0]))
    g1 = _n(np.cross(P1[1] - P1[0], P1[2] - P1[0]))
    # camera on the front side, within 70 deg of the shading normal
    for _ in range(100):
        w = _n(g1 + 0.8 * rng.normal(size=3))
        if np.dot(w, n1) > 0.35 and np.dot(w, g1) > 0.35:
            break
    x0 = x1 + rng.uniform(*dist) * w
    d0 = _n(x1 - x0)
    if chain[0] == "R":
        w1 = _reflect(d0, n1)
    else:
        w1 = _refract(d0, n1, eta_front, eta_back)
        if w1 is None:
            return None
    w1 = _n(w1)
    # the outgoing ray must leave on the correct side of both planes
    if chain[0] == "R" and not (np.dot(w1, n1) > 0.05 and np.dot(w1, g1) > 0.05):
        return None
    if chain[0] == "T" and not (np.dot(w1, n1) < -0.05 and np.dot(w1, g1) < -0.05):
        return None
    if len(chain) == 1:
        xk1 = x1 + rng.uniform(*dist) * w1
        mesh = Mesh(P1.astype(np.float32), N1.astype(np.float32), np.array([[0, 1, 2]], np.uint32), eta_front, eta_back)
        return mesh, [0], x0, xk1, np.array([u1, v1])
    # ---- k = 2: T_2 around x_2 = x_1 + L w1, facing back toward x_1 for R, along w1 for T (exit)
    L = rng.uniform(0.5, 1.5)
    x2 = x1 + L * w1
    eta1 = eta_front if chain[0] == "R" else eta_back
    entry = chain[1] == "T" and eta1 == eta_front  # ray in the front medium enters the dielectric at T2
    if chain[1] == "R" or entry:
        nrm2 = _n(-w1 + 0.3 * rng.normal(size=3))  # facing x1
    else:
        nrm2 = _n(w1 + 0.3 * rng.normal(size=3))  # exit face: geometric normal points out of the glass
    P2, N2, uv2 = _tri_around(rng, x2, nrm2, size * 2, tilt, face)
    # move x2 to an interior point of T2 on the ray: intersect the ray with T2
    e1, e2 = P2[1] - P2[0], P2[2] - P2[0]
    Pv = np.cross(w1, e2)
    det = np.dot(e1, Pv)
    s = x1 - P2[0]
    u2 = np.dot(s, Pv) / det
    Q = np.cross(s, e1)
    v2 = np.dot(w1, Q) / det
    t = np.dot(e2, Q) / det
    if not (t > 0 and u2 > 0.02 and v2 > 0.02 and u2 + v2 < 0.98):
        return None
    x2 = x1 + t * w1
    n2 = _n(N2[0] + u2 * (N2[1] - N2[0]) + v2 * (N2[2] - N2[0]))
    g2 = _n(np.cross(e1, e2))
    if chain[1] == "R":
        w2 = _reflect(w1, n2)
        if not (np.dot(-w1, n2) * np.dot(w2, n2) > 0 and np.dot(-w1, g2) * np.dot(w2, g2) > 0 and np.dot(-w1, n2) * np.dot(-w1, g2) > 0):
            return None
    elif entry:
        # x1 on T2's front side (the medium eta1 = eta_front), transmitted into eta_back
        if np.dot(x1 - P2[0], g2) < 0:
            return None
        w2 = _refract(w1, n2, eta1, eta_back)
        if w2 is None:
            return None
        if not (np.dot(w2, n2) < -0.05 and np.dot(w2, g2) < -0.05):
            return None
    else:
        # x1 must be on T2's back side (inside the dielectric)
        if np.dot(x1 - P2[0], g2) > 0:
            return None
        w2 = _refract(w1, n2, eta1, eta_front)
        if w2 is None:
            return None
        if not (np.dot(w2, n2) > 0.05 and np.dot(w2, g2) > 0.05):
            return None
    xk1 = x2 + rng.uniform(*dist) * _n(w2)
    pos = np.concatenate([P1, P2]).astype(np.float32)
    nrm = np.concatenate([N1, N2]).astype(np.float32)
    mesh = Mesh(pos, nrm, np.array([[0, 1, 2], [3, 4, 5]], np.uint32), eta_front, eta_back)
    return mesh, [0, 1], x0, xk1, np.array([u1, v1, u2, v2])


def planted_many(seed, chain, n, **kw):
    rng = np.random.default_rng(seed)
    out = []
    tries = 0
    while len(out) < n and tries < 50 * n:
        tries += 1
        p = planted(rng, chain, **kw)
        if p is not None:
            out.append(p)
    return out
