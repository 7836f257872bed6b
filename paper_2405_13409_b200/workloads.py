"""Seeded synthetic inputs shaped like the paper's workloads.

This module is the ONLY code shared by the oracle side (tests, bench cpu_baseline) and
the CUDA side.  It builds meshes (float32 positions + per-vertex shading normals +
uint32 triangle indices) and query endpoints (float64 x_0, x_{k+1}); it holds none of
the method's arithmetic (no polynomials, no resultants, no path validation).

Workloads (PAPER.md:665-748 describe the paper's scenes; their data is not available,
so each is replaced by a synthetic scene of the same shape):

* C1 ``patch``  - 256-tri interpolated-normal mirror patch, 1 query, R (BASELINE configs[0]).
* C2 ``glints`` - 100,352-tri normal-mapped bumpy plane, 256x256 light samples, R
                  (BASELINE configs[1]; "glints" scenes).
* C3 ``pool``   - 199,712-tri water surface, 512x512 floor receivers, T
                  (BASELINE configs[2]; "Pool").
* C4 ``sphere`` - 5,120-tri icosphere dielectric, 128x128 receivers, TT (configs[3]).
* C5 ``shell``  - glass shell sweep, 1024x1024 receivers, TT (configs[4]).

Every generator takes a seed and is deterministic (numpy PCG64).
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np


@dataclass
class Mesh:
    pos: np.ndarray          # (V,3) float32
    nrm: np.ndarray          # (V,3) float32, shading normals (unit, consistently oriented)
    tri: np.ndarray          # (T,3) uint32, CCW => geometric normal e1 x e2 points to the front side
    eta_front: float = 1.0   # IOR on the side the geometric normal points to
    eta_back: float = 1.0

    @property
    def ntris(self) -> int:
        return int(self.tri.shape[0])

    @property
    def nverts(self) -> int:
        return int(self.pos.shape[0])


@dataclass
class Workload:
    name: str
    chain: str                       # "R", "T", "RR", "TT"
    mesh: Mesh
    endpoints: np.ndarray            # (Q,2,3) float64: x_0, x_{k+1}
    intensity: np.ndarray            # (Q,) float64 point-light intensity at x_{k+1}
    meta: dict = field(default_factory=dict)

    @property
    def nqueries(self) -> int:
        return int(self.endpoints.shape[0])

    def subset(self, idx) -> "Workload":
        idx = np.asarray(idx)
        return Workload(self.name, self.chain, self.mesh, np.ascontiguousarray(self.endpoints[idx]),
                        np.ascontiguousarray(self.intensity[idx]), dict(self.meta, subset=len(idx)))


# ----------------------------------------------------------------------------- grids

def grid_mesh(nx: int, ny: int, x0: float, x1: float, y0: float, y1: float,
              height, grad) -> Mesh:
    """Regular (nx x ny)-vertex height-field grid, two CCW triangles per quad.

    ``height(x,y)`` gives z, ``grad(x,y)`` gives (dz/dx, dz/dy) of the SHADING surface;
    the shading normal is normalize(-dz/dx, -dz/dy, 1).
    """
    xs = np.linspace(x0, x1, nx)
    ys = np.linspace(y0, y1, ny)
    X, Y = np.meshgrid(xs, ys, indexing="xy")          # (ny, nx)
    Z = height(X, Y)
    gx, gy = grad(X, Y)
    N = np.stack([-gx, -gy, np.ones_like(gx)], axis=-1)
    N /= np.linalg.norm(N, axis=-1, keepdims=True)
    pos = np.stack([X, Y, Z], axis=-1).reshape(-1, 3).astype(np.float32)
    nrm = N.reshape(-1, 3).astype(np.float32)
    j, i = np.meshgrid(np.arange(ny - 1), np.arange(nx - 1), indexing="ij")
    v00 = (j * nx + i).ravel()
    v10 = v00 + 1
    v01 = v00 + nx
    v11 = v01 + 1
    t0 = np.stack([v00, v10, v11], axis=1)
    t1 = np.stack([v00, v11, v01], axis=1)
    tri = np.stack([t0, t1], axis=1).reshape(-1, 3).astype(np.uint32)
    return Mesh(pos, nrm, tri)


def _waves(rng, n: int, lam_lo: float, lam_hi: float):
    lam = rng.uniform(lam_lo, lam_hi, n)
    ang = rng.uniform(0, 2 * np.pi, n)
    k = (2 * np.pi / lam)[:, None] * np.stack([np.cos(ang), np.sin(ang)], axis=1)
    phi = rng.uniform(0, 2 * np.pi, n)
    return k, phi


def _wave_fields(A, k, phi):
    def height(X, Y):
        Z = np.zeros_like(X)
        for a, kk, p in zip(A, k, phi):
            Z += a * np.sin(kk[0] * X + kk[1] * Y + p)
        return Z

    def grad(X, Y):
        gx = np.zeros_like(X)
        gy = np.zeros_like(X)
        for a, kk, p in zip(A, k, phi):
            c = a * np.cos(kk[0] * X + kk[1] * Y + p)
            gx += c * kk[0]
            gy += c * kk[1]
        return gx, gy

    return height, grad


# ----------------------------------------------------------------------------- C1

def patch_c1() -> Workload:
    """C1: 17x9-vertex grid over [-1,1]x[-0.5,0.5], z = 0.05 sin(3x) cos(4y), analytic normals."""
    height = lambda X, Y: 0.05 * np.sin(3 * X) * np.cos(4 * Y)
    grad = lambda X, Y: (0.15 * np.cos(3 * X) * np.cos(4 * Y), -0.2 * np.sin(3 * X) * np.sin(4 * Y))
    mesh = grid_mesh(17, 9, -1.0, 1.0, -0.5, 0.5, height, grad)
    ep = np.array([[[0.0, -1.5, 1.0], [0.3, 1.2, 1.4]]], dtype=np.float64)
    return Workload("patch", "R", mesh, ep, np.ones(1), {"config": "C1"})


# ----------------------------------------------------------------------------- C2

def glints_c2(res: int = 256, nverts_side: int = 225, seed_bump: int = 1, seed_strata: int = 2) -> Workload:
    """C2: flat plane z=0 over [-1,1]^2 with a normal-mapped bump field (48 waves, RMS slope 0.2).

    Queries: x_0 = pinhole camera (0,-2,1.5); x_2 = stratified sample on a 0.2x0.2 area light
    centred at (0.5,1.0,2.0); pixel p -> stratum perm[p] (fixed permutation), jittered.
    """
    rng = np.random.default_rng(seed_bump)
    nwaves = 48
    k, phi = _waves(rng, nwaves, 0.02, 0.5)
    A = 1.0 / np.linalg.norm(k, axis=1)          # equal slope per wave before scaling
    A *= rng.uniform(0.5, 1.0, nwaves)
    _, grad = _wave_fields(A, k, phi)
    xs = np.linspace(-1, 1, 129)
    gx, gy = grad(*np.meshgrid(xs, xs))
    A *= 0.2 / np.sqrt(np.mean(gx ** 2 + gy ** 2))
    _, grad = _wave_fields(A, k, phi)
    mesh = grid_mesh(nverts_side, nverts_side, -1.0, 1.0, -1.0, 1.0, lambda X, Y: np.zeros_like(X), grad)

    rs = np.random.default_rng(seed_strata)
    Q = res * res
    perm = rs.permutation(Q)
    jit = rs.uniform(0, 1, (Q, 2))
    si = perm % res
    sj = perm // res
    lx = 0.5 + 0.2 * ((si + jit[:, 0]) / res - 0.5)
    ly = 1.0 + 0.2 * ((sj + jit[:, 1]) / res - 0.5)
    ep = np.zeros((Q, 2, 3))
    ep[:, 0] = (0.0, -2.0, 1.5)
    ep[:, 1, 0] = lx
    ep[:, 1, 1] = ly
    ep[:, 1, 2] = 2.0
    return Workload("glints", "R", mesh, ep, np.ones(Q), {"config": "C2", "res": res})


# ----------------------------------------------------------------------------- C3

def pool_c3(res: int = 512, nverts_side: int = 317, seed: int = 3) -> Workload:
    """C3: water surface z = sum_k A_k sin(k_k.(x,y)+phi_k) over [-1,1]^2, receivers on z=-1.

    Geometric normal points up (+z, air side, eta 1.0); the water side is eta 1.33.
    """
    rng = np.random.default_rng(seed)
    A = rng.uniform(0.002, 0.008, 4)
    k, phi = _waves(rng, 4, 0.2, 0.6)
    height, grad = _wave_fields(A, k, phi)
    mesh = grid_mesh(nverts_side, nverts_side, -1.0, 1.0, -1.0, 1.0, height, grad)
    mesh.eta_front, mesh.eta_back = 1.0, 1.33
    xs = -1.0 + (np.arange(res) + 0.5) * (2.0 / res)
    X, Y = np.meshgrid(xs, xs, indexing="xy")
    Q = res * res
    ep = np.zeros((Q, 2, 3))
    ep[:, 0, 0] = X.ravel()
    ep[:, 0, 1] = Y.ravel()
    ep[:, 0, 2] = -1.0
    ep[:, 1] = (0.2, 0.3, 2.0)
    return Workload("pool", "T", mesh, ep, np.ones(Q), {"config": "C3", "res": res})


# ----------------------------------------------------------------------------- spheres

def icosphere(level: int, radius: float = 1.0, inward: bool = False) -> Mesh:
    t = (1.0 + 5 ** 0.5) / 2
    v = [(-1, t, 0), (1, t, 0), (-1, -t, 0), (1, -t, 0), (0, -1, t), (0, 1, t), (0, -1, -t), (0, 1, -t),
         (t, 0, -1), (t, 0, 1), (-t, 0, -1), (-t, 0, 1)]
    f = [(0, 11, 5), (0, 5, 1), (0, 1, 7), (0, 7, 10), (0, 10, 11), (1, 5, 9), (5, 11, 4), (11, 10, 2),
         (10, 7, 6), (7, 1, 8), (3, 9, 4), (3, 4, 2), (3, 2, 6), (3, 6, 8), (3, 8, 9), (4, 9, 5), (2, 4, 11),
         (6, 2, 10), (8, 6, 7), (9, 8, 1)]
    verts = [np.array(p, float) / np.linalg.norm(p) for p in v]
    for _ in range(level):
        cache = {}
        nf = []

        def mid(a, b):
            key = (min(a, b), max(a, b))
            if key not in cache:
                m = verts[a] + verts[b]
                verts.append(m / np.linalg.norm(m))
                cache[key] = len(verts) - 1
            return cache[key]

        for a, b, c in f:
            ab, bc, ca = mid(a, b), mid(b, c), mid(c, a)
            nf += [(a, ab, ca), (b, bc, ab), (c, ca, bc), (ab, bc, ca)]
        f = nf
    P = np.array(verts)
    tri = np.array(f, dtype=np.uint32)
    N = P.copy()
    if inward:
        tri = tri[:, [0, 2, 1]]
        N = -N
    return Mesh((P * radius).astype(np.float32), N.astype(np.float32), np.ascontiguousarray(tri))


def merge(*meshes: Mesh) -> Mesh:
    pos, nrm, tri, off = [], [], [], 0
    for m in meshes:
        pos.append(m.pos)
        nrm.append(m.nrm)
        tri.append(m.tri + off)
        off += m.nverts
    return Mesh(np.concatenate(pos), np.concatenate(nrm), np.concatenate(tri).astype(np.uint32),
                meshes[0].eta_front, meshes[0].eta_back)


def sphere_c4(res: int = 128, level: int = 4) -> Workload:
    """C4: dielectric icosphere r=0.5 (level 4: 5,120 tris), receivers z=-1.5 over [-1,1]^2, light (0,0,3)."""
    mesh = icosphere(level, 0.5)
    mesh.eta_front, mesh.eta_back = 1.0, 1.5
    xs = -1.0 + (np.arange(res) + 0.5) * (2.0 / res)
    X, Y = np.meshgrid(xs, xs, indexing="xy")
    Q = res * res
    ep = np.zeros((Q, 2, 3))
    ep[:, 0, 0] = X.ravel()
    ep[:, 0, 1] = Y.ravel()
    ep[:, 0, 2] = -1.5
    ep[:, 1] = (0.0, 0.0, 3.0)
    return Workload("sphere", "TT", mesh, ep, np.ones(Q), {"config": "C4", "res": res})


def shell_c5(res: int = 1024, level: int = 3) -> Workload:
    """C5: glass shell (outer r=0.5, inner r=0.45 inward-facing), light inside the cavity,
    receivers on the wall y=2 over [-2,2]^2 (x,z)."""
    outer = icosphere(level, 0.5)
    inner = icosphere(level, 0.45, inward=True)
    mesh = merge(outer, inner)
    mesh.eta_front, mesh.eta_back = 1.0, 1.5
    xs = -2.0 + (np.arange(res) + 0.5) * (4.0 / res)
    X, Z = np.meshgrid(xs, xs, indexing="xy")
    Q = res * res
    ep = np.zeros((Q, 2, 3))
    ep[:, 0, 0] = X.ravel()
    ep[:, 0, 1] = 2.0
    ep[:, 0, 2] = Z.ravel()
    ep[:, 1] = (0.05, 0.02, 0.0)
    return Workload("shell", "TT", mesh, ep, np.ones(Q), {"config": "C5", "res": res})


def mirrors_rr(res: int = 64, quads: int = 128, seed: int = 5) -> Workload:
    """C5 RR variant: two facing bumpy mirror panels 1 m apart (x = -0.5 facing +x,
    x = +0.5 facing -x; y, z in [-0.5, 0.5]; quads x quads each), point light between them at
    (0, 0.2, 0), receivers on the wall y = -1.5 over x, z in [-1, 1]."""
    rng = np.random.default_rng(seed)
    k, phi = _waves(rng, 16, 0.05, 0.5)
    A = 0.2 / np.linalg.norm(k, axis=1) / 4.0
    _, grad = _wave_fields(A, k, phi)
    base = grid_mesh(quads + 1, quads + 1, -0.5, 0.5, -0.5, 0.5, lambda X, Y: np.zeros_like(X), grad)
    # panel A: (x, y) grid -> world (x=-0.5, y=X, z=Y), normal (nz, nx, ny) facing +x
    def place(m, sign):
        P = m.pos.astype(np.float64)
        N = m.nrm.astype(np.float64)
        pos = np.stack([np.full(len(P), -0.5 * sign), P[:, 0], P[:, 1]], 1)
        nrm = np.stack([sign * N[:, 2], N[:, 0], N[:, 1]], 1)
        tri = m.tri.copy()
        # winding: geometric normal must face the other panel (+x for A, -x for B)
        p = pos[tri]
        g = np.cross(p[:, 1] - p[:, 0], p[:, 2] - p[:, 0])
        flip = g[:, 0] * sign < 0
        tri[flip] = tri[flip][:, [0, 2, 1]]
        return Mesh(pos.astype(np.float32), nrm.astype(np.float32), tri.astype(np.uint32))
    mesh = merge(place(base, 1.0), place(base, -1.0))
    xs = -1.0 + (np.arange(res) + 0.5) * (2.0 / res)
    X, Z = np.meshgrid(xs, xs, indexing="xy")
    Q = res * res
    ep = np.zeros((Q, 2, 3))
    ep[:, 0, 0] = X.ravel()
    ep[:, 0, 1] = -1.5
    ep[:, 0, 2] = Z.ravel()
    ep[:, 1] = (0.0, 0.2, 0.0)
    return Workload("mirrors", "RR", mesh, ep, np.ones(Q), {"config": "C5-RR", "res": res})


def random_triangles(rng, n: int, size: float, center=(0.0, 0.0, 0.0), spread: float = 1.0,
                     normal_tilt: float = 0.2, face: bool = False) -> Mesh:
    """Independent random triangles (for parity fuzzing): roughly facing +z, random vertex-normal tilt."""
    c = np.asarray(center) + rng.uniform(-spread, spread, (n, 3)) * np.array([1, 1, 0.2])
    P = c[:, None, :] + size * rng.normal(size=(n, 3, 3)) * np.array([1, 1, 0.2])
    e1 = P[:, 1] - P[:, 0]
    e2 = P[:, 2] - P[:, 0]
    g = np.cross(e1, e2)
    flip = g[:, 2] < 0
    P[flip] = P[flip][:, [0, 2, 1]]
    g = np.cross(P[:, 1] - P[:, 0], P[:, 2] - P[:, 0])
    g /= np.linalg.norm(g, axis=1, keepdims=True)
    if face:
        N = np.repeat(g[:, None, :], 3, axis=1)
    else:
        N = g[:, None, :] + normal_tilt * rng.normal(size=(n, 3, 3))
        N /= np.linalg.norm(N, axis=2, keepdims=True)
    pos = P.reshape(-1, 3).astype(np.float32)
    nrm = N.reshape(-1, 3).astype(np.float32)
    tri = np.arange(3 * n, dtype=np.uint32).reshape(n, 3)
    return Mesh(pos, nrm, tri)


CONFIGS = {
    "C1": patch_c1,
    "C2": glints_c2,
    "C3": pool_c3,
    "C4": sphere_c4,
    "C5": shell_c5,
    "C5RR": mirrors_rr,
}


# ----------------------------------------------------------------------------- glossy + renderer inputs

def beckmann_slopes(seed: int, nsamples: int, ntris: int, alpha: float) -> np.ndarray:
    """Microfacet slope samples for the glossy extension (reading R28): Beckmann slopes p, q are
    independent N(0, alpha^2 / 2).  Returns (nsamples, ntris, 2) float64 (the random numbers the method draws,
    passed to both sides as inputs)."""
    rng = np.random.default_rng(seed)
    return rng.normal(0.0, alpha / np.sqrt(2.0), size=(nsamples, ntris, 2))


MIRROR_LIGHT = (0.1, -0.05, 0.5)


def mirror_caustic(res: int = 128, half: float = 1.5) -> Workload:
    """Renderer fixture ("flat-mirror caustic line fixture"): one face-normal mirror triangle in the plane
    z = 1 facing down (normals (0,0,-1)), a point light at MIRROR_LIGHT below it, and res x res receivers at the pixel
    centres of [-half, half]^2 on z = 0 (row-major, x fastest).  Chain R (x_0 = receiver, x_2 = light)."""
    pos = np.array([[-0.21, -0.175, 1.0], [0.0, 0.2275, 1.0], [0.245, -0.105, 1.0]], np.float32)
    nrm = np.tile([0.0, 0.0, -1.0], (3, 1)).astype(np.float32)
    mesh = Mesh(pos, nrm, np.array([[0, 1, 2]], np.uint32))
    c = -half + (np.arange(res) + 0.5) * (2 * half / res)
    X, Y = np.meshgrid(c, c)
    x0 = np.stack([X.ravel(), Y.ravel(), np.zeros(res * res)], 1)
    ep = np.stack([x0, np.tile(np.array(MIRROR_LIGHT), (res * res, 1))], 1)
    return Workload("mirror_caustic", "R", mesh, np.ascontiguousarray(ep), np.ones(res * res), {"res": res})
