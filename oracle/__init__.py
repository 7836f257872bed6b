"""ORACLE — test infrastructure only.

Python wrapper (ctypes) around the plain C++ FP64 oracle in oracle/oracle.cpp.  Only tests/,
__graft_entry__.smoke() and bench.py (cpu_baseline / --impl reference) may import this package.
The product path (paper_2405_13409_b200) never imports it and shares no code with it.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "liboracle.so")
SRCS = [os.path.join(HERE, "oracle.cpp")]
DEPS = SRCS + [os.path.join(HERE, "poly.hpp"), os.path.join(HERE, "oracle.h")]

FLAG_NEAR_TANGENT = 1
FLAG_BOUNDARY = 2
FLAG_RESIDUAL = 4
FLAG_DEGENERATE = 8

_lock = threading.Lock()
_lib = None


def build(force: bool = False) -> str:
    """Compile liboracle.so with g++ (plain -O2, no fast-math: the oracle is the reference)."""
    stale = force or not os.path.exists(LIB) or any(os.path.getmtime(d) > os.path.getmtime(LIB) for d in DEPS)
    if stale:
        cmd = ["g++", "-O2", "-std=c++17", "-fPIC", "-shared", "-pthread", "-o", LIB + ".tmp"] + SRCS
        subprocess.check_call(cmd, cwd=HERE)
        os.replace(LIB + ".tmp", LIB)
    return LIB


class Config(ctypes.Structure):
    _fields_ = [("pieces", ctypes.c_int), ("scan_bisect_iters", ctypes.c_int), ("bisect_tol", ctypes.c_double),
                ("polish_iters", ctypes.c_int), ("theta_admit", ctypes.c_double), ("theta_final", ctypes.c_double),
                ("eps_domain", ctypes.c_double), ("eps_flag", ctypes.c_double), ("tau_trunc", ctypes.c_double),
                ("cull", ctypes.c_int), ("cull_margin", ctypes.c_double),
                ("cull_levels", ctypes.c_int), ("visibility", ctypes.c_int)]


def lib():
    global _lib
    with _lock:
        if _lib is None:
            build()
            L = ctypes.CDLL(LIB)
            P = ctypes.c_void_p
            L.orc_solve.restype = P
            L.orc_solve.argtypes = [P, P, ctypes.c_uint32, P, ctypes.c_uint32, ctypes.c_float, ctypes.c_float,
                                    ctypes.c_char_p, P, ctypes.c_uint32, P, P, P, P, ctypes.c_int, P,
                                    ctypes.c_uint32, P, ctypes.c_uint32]
            L.orc_free.argtypes = [P]
            for f in ("orc_n_solutions", "orc_n_flagged"):
                getattr(L, f).restype = ctypes.c_uint64
                getattr(L, f).argtypes = [P]
            L.orc_k.argtypes = [P]
            L.orc_get_solutions.argtypes = [P] * 7
            L.orc_get_flagged.argtypes = [P] * 4
            L.orc_get_per_query.argtypes = [P, P]
            L.orc_get_report.argtypes = [P, P]
            L.orc_n_worklist.restype = ctypes.c_uint64
            L.orc_n_worklist.argtypes = [P]
            L.orc_get_worklist.argtypes = [P, P, P]
            L.orc_default_config.argtypes = [P]
            L.orc_build_system.argtypes = [ctypes.c_char_p, P, P, P, ctypes.c_double, ctypes.c_double, P, P, P, P,
                                           P, P]
            L.orc_bezout.argtypes = [P, ctypes.c_int, P, ctypes.c_int, ctypes.c_int, P, P]
            L.orc_det_laplace.argtypes = [P, P, ctypes.c_int, P]
            L.orc_det_at.restype = ctypes.c_double
            L.orc_det_at.argtypes = [P, ctypes.c_int, P, ctypes.c_int, ctypes.c_int, ctypes.c_double]
            L.orc_isolate.argtypes = [P, ctypes.c_int, ctypes.c_double, ctypes.c_double, ctypes.c_double, P]
            L.orc_cull_keep.argtypes = [ctypes.c_char_p, P, P, P, ctypes.c_double, ctypes.c_double, ctypes.c_double,
                                        ctypes.c_int]
            L.orc_jacobian.restype = ctypes.c_double
            L.orc_jacobian.argtypes = [ctypes.c_char_p, P, P, P, ctypes.c_double, ctypes.c_double, P]
            L.orc_sqrt_table.argtypes = [P]
            L.orc_sqrt_approx.restype = ctypes.c_double
            L.orc_sqrt_approx.argtypes = [ctypes.c_double]
            _lib = L
    return _lib


def _p(a):
    return a.ctypes.data_as(ctypes.c_void_p) if a is not None else None


def default_config(**kw) -> Config:
    c = Config()
    lib().orc_default_config(ctypes.byref(c))
    for k, v in kw.items():
        setattr(c, k, v)
    return c


class Result:
    """Solutions sorted by (query, tuple order in the list, root order)."""

    def __init__(self, k, query, tuple_, bary, contribution, residual, flags, fq, ftup, fflags, per_query, report):
        self.k = k
        self.query = query
        self.tuple = tuple_
        self.bary = bary
        self.contribution = contribution
        self.residual = residual
        self.flags = flags
        self.flagged_query = fq
        self.flagged_tuple = ftup
        self.flagged_flags = fflags
        self.per_query = per_query
        self.report = report

    @property
    def n_solutions(self):
        return int(self.query.shape[0])


REPORT_KEYS = ["pairs_in", "systems", "vroots", "candidates", "rej_domain", "rej_constraint", "rej_side",
               "rej_kappa", "flagged", "admissible", "rej_visibility"]


def solve(mesh, chain: str, endpoints: np.ndarray, intensity=None, offsets=None, tri_ids=None, cfg: Config = None,
          nthreads: int = 0, occluders=None) -> Result:
    """occluders: optional non-specular Mesh blocking segments when cfg.visibility."""
    L = lib()
    pos = np.ascontiguousarray(mesh.pos, dtype=np.float32)
    nrm = np.ascontiguousarray(mesh.nrm, dtype=np.float32)
    tri = np.ascontiguousarray(mesh.tri, dtype=np.uint32)
    ep = np.ascontiguousarray(endpoints, dtype=np.float64)
    nq = ep.shape[0]
    inten = None if intensity is None else np.ascontiguousarray(intensity, dtype=np.float64)
    off = None if offsets is None else np.ascontiguousarray(offsets, dtype=np.uint32)
    ids = None if tri_ids is None else np.ascontiguousarray(tri_ids, dtype=np.uint32)
    cfg = cfg or default_config()
    opos = otri = None
    if occluders is not None:
        opos = np.ascontiguousarray(occluders.pos, dtype=np.float32)
        otri = np.ascontiguousarray(occluders.tri, dtype=np.uint32)
    h = L.orc_solve(_p(pos), _p(nrm), pos.shape[0], _p(tri), tri.shape[0], mesh.eta_front, mesh.eta_back,
                    chain.encode(), _p(ep), nq, _p(inten), _p(off), _p(ids), ctypes.byref(cfg), nthreads,
                    _p(opos), 0 if opos is None else opos.shape[0], _p(otri), 0 if otri is None else otri.shape[0])
    if not h:
        raise ValueError("oracle rejected the input")
    try:
        k = len(chain)
        n = L.orc_n_solutions(h)
        m = L.orc_n_flagged(h)
        q = np.zeros(n, np.uint32)
        t = np.zeros(n * k, np.uint32)
        b = np.zeros(n * 2 * k, np.float64)
        c = np.zeros(n, np.float64)
        r = np.zeros(n, np.float64)
        f = np.zeros(n, np.uint32)
        L.orc_get_solutions(h, _p(q), _p(t), _p(b), _p(c), _p(r), _p(f))
        fq = np.zeros(m, np.uint32)
        ft = np.zeros(m * k, np.uint32)
        ff = np.zeros(m, np.uint32)
        L.orc_get_flagged(h, _p(fq), _p(ft), _p(ff))
        pq = np.zeros(nq, np.float64)
        L.orc_get_per_query(h, _p(pq))
        rep = np.zeros(11, np.uint64)
        L.orc_get_report(h, _p(rep))
        nw = L.orc_n_worklist(h)
        wq = np.zeros(nw, np.uint32)
        wt = np.zeros(nw * k, np.uint32)
        L.orc_get_worklist(h, _p(wq), _p(wt))
    finally:
        L.orc_free(h)
    res = Result(k, q, t.reshape(n, k), b.reshape(n, 2 * k), c, r, f, fq, ft.reshape(m, k), ff, pq,
                 dict(zip(REPORT_KEYS, (int(x) for x in rep))))
    res.worklist = (wq, wt.reshape(nw, k))  # the (query, tuple) pairs the oracle solved (after its cull)
    return res


def tri_block(mesh, ids) -> np.ndarray:
    """(k*18,) float64 block (p0,p1,p2,n0,n1,n2) per triangle, original labeling."""
    out = []
    for t in np.atleast_1d(ids):
        vi = mesh.tri[int(t)]
        out.append(np.concatenate([mesh.pos[vi].astype(np.float64).ravel(), mesh.nrm[vi].astype(np.float64).ravel()]))
    return np.concatenate(out)


def build_system(chain, tris18: np.ndarray, x0, xk1, eta_front=1.0, eta_back=1.0):
    """Returns (a, b, info) with a, b dense (deg+1)^2 coefficient grids [i, j] = coeff of u^i v^j."""
    L = lib()
    a = np.zeros(64 * 64)
    b = np.zeros(64 * 64)
    da = ctypes.c_int()
    db = ctypes.c_int()
    info = np.zeros(3, np.int32)
    t = np.ascontiguousarray(tris18, dtype=np.float64)
    x0 = np.ascontiguousarray(x0, dtype=np.float64)
    xk1 = np.ascontiguousarray(xk1, dtype=np.float64)
    rc = L.orc_build_system(chain.encode(), _p(t), _p(x0), _p(xk1), eta_front, eta_back, None, _p(a),
                            ctypes.byref(da), _p(b), ctypes.byref(db), _p(info))
    if rc != 0:
        raise ValueError("bad chain")
    A = a[:(da.value + 1) ** 2].reshape(da.value + 1, da.value + 1).copy()
    B = b[:(db.value + 1) ** 2].reshape(db.value + 1, db.value + 1).copy()
    return A, B, {"relabel": int(info[0]), "eta0": info[1] / 1000.0, "degenerate_basis": int(info[2])}


def bezout(A: np.ndarray, B: np.ndarray, n: int):
    """Bezout matrix (Eq. 24) with polynomial entries: list of lists of coefficient arrays."""
    L = lib()
    A = np.ascontiguousarray(A, dtype=np.float64)
    B = np.ascontiguousarray(B, dtype=np.float64)
    ent = np.zeros(n * n * 128)
    deg = np.zeros(n * n, np.int32)
    L.orc_bezout(_p(A), A.shape[0] - 1, _p(B), B.shape[0] - 1, n, _p(ent), _p(deg))
    ent = ent.reshape(n, n, 128)
    return [[ent[i, j, :deg[i * n + j] + 1].copy() for j in range(n)] for i in range(n)]


def det_laplace(M):
    L = lib()
    n = len(M)
    ent = np.zeros(n * n * 128)
    deg = np.zeros(n * n, np.int32)
    for i in range(n):
        for j in range(n):
            c = np.asarray(M[i][j], dtype=np.float64)
            ent[(i * n + j) * 128:(i * n + j) * 128 + len(c)] = c
            deg[i * n + j] = len(c) - 1
    out = np.zeros(4096)
    d = L.orc_det_laplace(_p(ent), _p(deg), n, _p(out))
    return out[:d + 1].copy()


def det_at(A, B, n, v):
    L = lib()
    A = np.ascontiguousarray(A, dtype=np.float64)
    B = np.ascontiguousarray(B, dtype=np.float64)
    return L.orc_det_at(_p(A), A.shape[0] - 1, _p(B), B.shape[0] - 1, n, v)


def isolate(p, lo=0.0, hi=1.0, tol=1e-9):
    L = lib()
    p = np.ascontiguousarray(p, dtype=np.float64)
    out = np.zeros(max(len(p), 1) * 4)
    n = L.orc_isolate(_p(p), len(p) - 1, lo, hi, tol, _p(out))
    return out[:n].copy()


def cull_keep(chain, tris18, x0, xk1, eta_front=1.0, eta_back=1.0, margin=1e-9, levels=3) -> bool:
    L = lib()
    t = np.ascontiguousarray(tris18, dtype=np.float64)
    x0 = np.ascontiguousarray(x0, dtype=np.float64)
    xk1 = np.ascontiguousarray(xk1, dtype=np.float64)
    return bool(L.orc_cull_keep(chain.encode(), _p(t), _p(x0), _p(xk1), eta_front, eta_back, margin, levels))


def jacobian(chain, tris18, x0, xk1, bary, eta_front=1.0, eta_back=1.0) -> float:
    L = lib()
    t = np.ascontiguousarray(tris18, dtype=np.float64)
    x0 = np.ascontiguousarray(x0, dtype=np.float64)
    xk1 = np.ascontiguousarray(xk1, dtype=np.float64)
    b = np.ascontiguousarray(bary, dtype=np.float64)
    return L.orc_jacobian(chain.encode(), _p(t), _p(x0), _p(xk1), eta_front, eta_back, _p(b))


def sqrt_table() -> np.ndarray:
    out = np.zeros(30)
    lib().orc_sqrt_table(_p(out))
    return out.reshape(6, 5)


def sqrt_approx(x: float) -> float:
    return lib().orc_sqrt_approx(float(x))


# ----------------------------------------------------------------------------- glossy vertices + splat renderer

class MeshArrays:
    """Plain container with the attributes solve() reads (pos, nrm, tri, eta_front, eta_back)."""

    def __init__(self, pos, nrm, tri, eta_front=1.0, eta_back=1.0):
        self.pos, self.nrm, self.tri = pos, nrm, tri
        self.eta_front, self.eta_back = eta_front, eta_back


def perturb_normals(mesh, slopes: np.ndarray) -> MeshArrays:
    """Glossy vertices: "After sampling the normal offset for glossy vertices, the admissible chains
    corresponding to the offset remain finite, and the problem reduces to pure specular situations."
    reading R28: triangle t's three shading normals get the offset p_t T_t + q_t B_t, with T_t = e1 / |e1| and
    B_t = g^ x T_t (g = e1 x e2) the orthonormal frame of its plane, n_j' = fl32(n_j + p T + q B) in FP64.
    slopes: (ntris, 2) float64.  Returns a de-indexed mesh (three own vertices per triangle, same triangle ids) so
    that shared vertices can carry each triangle's own normal.  Pinned by tests/test_glossy_render.py (frame
    properties, tilt angle, zero-offset identity, brute-force shooting on the perturbed surface)."""
    tri = np.asarray(mesh.tri, dtype=np.int64)
    P = np.asarray(mesh.pos, dtype=np.float32)[tri].astype(np.float64)      # (T, 3, 3)
    N = np.asarray(mesh.nrm, dtype=np.float32)[tri].astype(np.float64)
    s = np.asarray(slopes, dtype=np.float64).reshape(len(tri), 2)
    e1 = P[:, 1] - P[:, 0]
    e2 = P[:, 2] - P[:, 0]
    g = np.cross(e1, e2)
    gh = g / np.sqrt(np.sum(g * g, axis=1))[:, None]
    T = e1 / np.sqrt(np.sum(e1 * e1, axis=1))[:, None]
    B = np.cross(gh, T)
    h = s[:, 0:1] * T + s[:, 1:2] * B
    N2 = (N + h[:, None, :]).astype(np.float32)
    pos = P.astype(np.float32).reshape(-1, 3)
    return MeshArrays(pos, N2.reshape(-1, 3), np.arange(3 * len(tri), dtype=np.uint32).reshape(-1, 3),
                      mesh.eta_front, mesh.eta_back)


def tonemap_srgb(radiance: np.ndarray, exposure: float = 1.0) -> np.ndarray:
    """8-bit gamma-2.2 gray code ("binary PPM (P6, 8-bit, sRGB with gamma 2.2)"):
    c = rint(255 * min(1, max(0, exposure * L))^(1/2.2)), replicated over 3 channels."""
    v = np.minimum(1.0, np.maximum(0.0, exposure * np.asarray(radiance, dtype=np.float64)))
    c = np.rint(255.0 * v ** (1.0 / 2.2)).astype(np.uint8)
    return np.repeat(c[..., None], 3, axis=-1)


def render(mesh, chain: str, endpoints: np.ndarray, width: int, height: int, intensity=None, slopes=None,
           albedo: float = 1.0, exposure: float = 1.0, cfg: Config = None, nthreads: int = 0):
    """Deterministic splat renderer (SPEC S:661-669 cmd_render, no Monte Carlo): pixel q is query q
    (row-major); per offset sample s the chains are solved on the perturbed surface and
        radiance[q] = sum_s (albedo / pi / S) * per_query_s[q]   (samples in order).
    slopes: (S, ntris, 2) or None (one pure specular solve).  Returns (radiance (H, W), srgb (H, W, 3) uint8,
    [oracle Result per sample]).  Pinned by tests/test_glossy_render.py (image-source mask IoU = 1 and radiance
    albedo/pi * I / L^2 of a flat-mirror caustic, sample averaging, gamma codes of known values)."""
    S = 1 if slopes is None else int(np.asarray(slopes).shape[0])
    nq = width * height
    acc = np.zeros(nq)
    scale = albedo / np.pi / S
    results = []
    for s in range(S):
        m = mesh if slopes is None else perturb_normals(mesh, np.asarray(slopes)[s])
        r = solve(m, chain, endpoints, intensity, cfg=cfg, nthreads=nthreads)
        acc += scale * r.per_query
        results.append(r)
    return acc.reshape(height, width), tonemap_srgb(acc, exposure).reshape(height, width, 3), results
