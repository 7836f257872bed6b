"""Thin ctypes binding of libspoly.so with the names of include/spoly.h.

Argument marshalling only: every step of the hot path runs in the CUDA kernels behind the C-ABI.
Device inputs are torch CUDA tensors (their data_ptr()); device outputs are returned as zero-copy
torch views of the ctx-owned buffers (valid until the next solve / destroy; clone() to keep).
There is no CPU fallback: importing on a machine without the built library raises.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
# SPOLY_LIB: alternative build of the same library (A/B kernel variants); default the in-tree build
LIB_PATH = os.environ.get("SPOLY_LIB") or os.path.join(HERE, "libspoly.so")

SPOLY_OK = 0
STATUS = {0: "SPOLY_OK", 1: "SPOLY_ERR_INVALID_ARG", 2: "SPOLY_ERR_BAD_MESH", 3: "SPOLY_ERR_UNSUPPORTED_CHAIN",
          4: "SPOLY_ERR_OOM", 5: "SPOLY_ERR_CAPACITY", 6: "SPOLY_ERR_CUDA"}
FLAG_NEAR_TANGENT, FLAG_BOUNDARY, FLAG_RESIDUAL, FLAG_DEGENERATE, FLAG_TRUNCATED = 1, 2, 4, 8, 16

EXPORTS = ["spoly_default_config", "spoly_create", "spoly_destroy", "spoly_last_error", "spoly_upload_mesh",
           "spoly_solve", "spoly_solve_host", "spoly_last_worklist", "spoly_bench_fma", "spoly_sqrt_table", "spoly_upload_occluders",
           "spoly_set_normal_offsets", "spoly_render"]


class SpolyError(RuntimeError):
    pass


class spoly_config(ctypes.Structure):
    _fields_ = [("pieces", ctypes.c_int), ("scan_bisect_iters", ctypes.c_int), ("bisect_tol", ctypes.c_double),
                ("polish_iters", ctypes.c_int), ("theta_admit", ctypes.c_double), ("theta_final", ctypes.c_double),
                ("eps_domain", ctypes.c_double), ("eps_flag", ctypes.c_double), ("tau_trunc", ctypes.c_double),
                ("cull", ctypes.c_int), ("deterministic", ctypes.c_int), ("cull_margin", ctypes.c_float),
                ("max_solutions", ctypes.c_uint64), ("max_pairs", ctypes.c_uint64),
                ("cull_levels", ctypes.c_int), ("visibility", ctypes.c_int), ("scan_restrict", ctypes.c_int),
                ("k2_tiles", ctypes.c_int)]


class spoly_tuple_list(ctypes.Structure):
    _fields_ = [("offsets", ctypes.c_void_p), ("tri_ids", ctypes.c_void_p)]


REPORT_FIELDS = ["n_pairs_in", "n_systems", "n_vroots", "n_candidates", "n_rej_domain", "n_rej_constraint",
                 "n_rej_side", "n_rej_kappa", "n_flagged", "n_admissible"]


class spoly_report(ctypes.Structure):
    _fields_ = [(f, ctypes.c_uint64) for f in REPORT_FIELDS] + [
        ("ms_cull", ctypes.c_float), ("ms_solve", ctypes.c_float), ("ms_reduce", ctypes.c_float),
        ("n_launches", ctypes.c_uint32), ("n_eval_terms", ctypes.c_uint64), ("required_solutions", ctypes.c_uint64),
        ("ms_phase1", ctypes.c_float), ("ms_phase2", ctypes.c_float), ("n_rebuilds", ctypes.c_uint64),
        ("alg_kflop", ctypes.c_uint64), ("n_jobs_mono", ctypes.c_uint64), ("n_jobs_deep", ctypes.c_uint64),
        ("n_elims", ctypes.c_uint64), ("n_pairs_coarse", ctypes.c_uint64),
        ("ms_roots", ctypes.c_float), ("ms_path", ctypes.c_float), ("n_refined", ctypes.c_uint64),
        ("n_cand_jobs", ctypes.c_uint64), ("n_path_jobs", ctypes.c_uint64), ("n_cull_tests", ctypes.c_uint64),
        ("n_truncated", ctypes.c_uint64), ("n_big_scan", ctypes.c_uint64), ("n_eval_deep", ctypes.c_uint64),
        ("n_rej_visibility", ctypes.c_uint64)]


class spoly_result(ctypes.Structure):
    _fields_ = [("n_solutions", ctypes.c_uint64), ("n_flagged", ctypes.c_uint64), ("k", ctypes.c_int),
                ("query", ctypes.c_void_p), ("tuple", ctypes.c_void_p), ("bary", ctypes.c_void_p),
                ("contribution", ctypes.c_void_p), ("residual", ctypes.c_void_p), ("flags", ctypes.c_void_p),
                ("flagged_query", ctypes.c_void_p), ("flagged_tuple", ctypes.c_void_p),
                ("flagged_flags", ctypes.c_void_p), ("per_query", ctypes.c_void_p), ("report", spoly_report)]


_lib = None


def lib():
    """Load libspoly.so (must have been built by build.py / __graft_entry__.build())."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise SpolyError(f"{LIB_PATH} is missing: run `python -m paper_2405_13409_b200.build` "
                             "(there is no CPU fallback)")
        L = ctypes.CDLL(LIB_PATH)
        P, I, U32, U64, D = ctypes.c_void_p, ctypes.c_int, ctypes.c_uint32, ctypes.c_uint64, ctypes.c_double
        L.spoly_default_config.argtypes = [P]
        L.spoly_create.argtypes = [I, P, P, P]
        L.spoly_destroy.argtypes = [P]
        L.spoly_destroy.restype = None
        L.spoly_last_error.argtypes = [P]
        L.spoly_last_error.restype = ctypes.c_char_p
        L.spoly_upload_mesh.argtypes = [P, P, P, U32, P, U32, ctypes.c_float, ctypes.c_float, P]
        L.spoly_solve.argtypes = [P, U32, ctypes.c_char_p, I, P, U32, P, P, P]
        L.spoly_solve_host.argtypes = [P, U32, ctypes.c_char_p, I, P, U32, P, P, P]
        L.spoly_last_worklist.argtypes = [P, P, P, P]
        L.spoly_bench_fma.argtypes = [P, I, D, P]
        L.spoly_sqrt_table.argtypes = [P, I, P]
        L.spoly_upload_occluders.argtypes = [P, P, U32, P, U32]
        L.spoly_set_normal_offsets.argtypes = [P, P, U32]
        L.spoly_render.argtypes = [P, U32, ctypes.c_char_p, I, P, U32, U32, P, U32, P, D, D, P, P]
        _lib = L
    return _lib


def sqrt_table(ctx=None) -> np.ndarray:
    """The Eq. 20 sqrt-surrogate table compiled into the library (6 x 5): the host copy (ctx None) or the
    device's constant-memory copy (ctx a Context)."""
    out = np.zeros(30, np.float64)
    h = ctx._h if ctx is not None else None
    rc = lib().spoly_sqrt_table(h, 1 if ctx is not None else 0, out.ctypes.data)
    if rc != SPOLY_OK:
        raise SpolyError(f"spoly_sqrt_table: {STATUS.get(rc, rc)}")
    return out.reshape(6, 5)


def default_config(**kw) -> spoly_config:
    c = spoly_config()
    lib().spoly_default_config(ctypes.byref(c))
    for k, v in kw.items():
        setattr(c, k, v)
    return c


class _CudaArray:
    """__cuda_array_interface__ shim for zero-copy torch views of ctx-owned device memory."""

    def __init__(self, ptr, shape, typestr):
        self.__cuda_array_interface__ = {"data": (int(ptr or 0), False), "shape": tuple(shape), "typestr": typestr,
                                         "version": 3, "strides": None}


def _view(ptr, shape, typestr, device):
    import torch
    n = int(np.prod(shape)) if len(shape) else 1
    dt = {"<u4": torch.int32, "<f8": torch.float64, "<f4": torch.float32}[typestr]
    if n == 0 or not ptr:
        return torch.zeros(shape, dtype=dt, device=device)
    return torch.as_tensor(_CudaArray(ptr, shape, typestr), device=device)


@dataclass
class Result:
    """Device-side result (torch views).  query/tuple/flags are int32 views of uint32 data."""
    n_solutions: int
    n_flagged: int
    k: int
    query: object
    tuple: object
    bary: object
    contribution: object
    residual: object
    flags: object
    flagged_query: object
    flagged_tuple: object
    flagged_flags: object
    per_query: object
    report: dict

    def to_numpy(self):
        out = {}
        for f in ("query", "tuple", "bary", "contribution", "residual", "flags", "flagged_query", "flagged_tuple",
                  "flagged_flags", "per_query"):
            a = getattr(self, f).cpu().numpy()
            if a.dtype == np.int32:
                a = a.view(np.uint32)
            out[f] = a
        return out


class Context:
    """RAII wrapper of spoly_ctx (one per device / process)."""

    def __init__(self, device: int = 0, config: spoly_config = None, stream=None):
        self._L = lib()
        self.device = device
        h = ctypes.c_void_p()
        st = None
        if stream is not None:
            st = ctypes.c_void_p(int(stream.cuda_stream if hasattr(stream, "cuda_stream") else stream))
        rc = self._L.spoly_create(device, ctypes.byref(config) if config is not None else None, st, ctypes.byref(h))
        if rc != SPOLY_OK:
            raise SpolyError(f"spoly_create: {STATUS.get(rc, rc)}")
        self._h = h
        self.k = None
        self.nq = 0

    def _check(self, rc, what):
        if rc != SPOLY_OK:
            msg = self._L.spoly_last_error(self._h)
            raise SpolyError(f"{what}: {STATUS.get(rc, rc)}: {msg.decode() if msg else ''}")

    def close(self):
        if getattr(self, "_h", None):
            self._L.spoly_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    def upload_mesh(self, mesh) -> int:
        pos = np.ascontiguousarray(mesh.pos, dtype=np.float32)
        nrm = np.ascontiguousarray(mesh.nrm, dtype=np.float32)
        tri = np.ascontiguousarray(mesh.tri, dtype=np.uint32)
        mid = ctypes.c_uint32()
        rc = self._L.spoly_upload_mesh(self._h, pos.ctypes.data, nrm.ctypes.data, pos.shape[0], tri.ctypes.data,
                                       tri.shape[0], float(mesh.eta_front), float(mesh.eta_back), ctypes.byref(mid))
        self._check(rc, "spoly_upload_mesh")
        return mid.value

    def upload_occluders(self, mesh=None):
        """Occluder-only triangles for the visibility test (cfg.visibility); None removes them."""
        if mesh is None:
            self._check(self._L.spoly_upload_occluders(self._h, None, 0, None, 0), "spoly_upload_occluders")
            return
        pos = np.ascontiguousarray(mesh.pos, dtype=np.float32)
        tri = np.ascontiguousarray(mesh.tri, dtype=np.uint32)
        rc = self._L.spoly_upload_occluders(self._h, pos.ctypes.data, pos.shape[0], tri.ctypes.data, tri.shape[0])
        self._check(rc, "spoly_upload_occluders")

    def set_normal_offsets(self, slopes=None):
        """Glossy microfacet offsets (reading R28): slopes (ntris, 2) float64 numpy in original
        triangle order, or None to restore the uploaded normals."""
        if slopes is None:
            self._check(self._L.spoly_set_normal_offsets(self._h, None, 0), "spoly_set_normal_offsets")
            return
        sl = np.ascontiguousarray(slopes, dtype=np.float64)
        self._check(self._L.spoly_set_normal_offsets(self._h, sl.ctypes.data, sl.shape[0]),
                    "spoly_set_normal_offsets")

    def render(self, chain: str, endpoints, width: int, height: int, intensity=None, slopes=None, albedo=1.0,
               exposure=1.0, srgb: bool = True, mesh_id: int = 0):
        """Deterministic splat renderer (spoly_render).  endpoints: CUDA float64 (W*H, 2, 3), row-major pixels;
        slopes: numpy (S, ntris, 2) float64 or None.  Returns (radiance CUDA float64 (H, W), sRGB CUDA uint8
        (H, W, 3) or None)."""
        import torch
        assert endpoints.is_cuda and endpoints.dtype == torch.float64 and endpoints.is_contiguous()
        nq = width * height
        assert endpoints.shape[0] == nq
        dev = endpoints.device
        rad = torch.empty(nq, dtype=torch.float64, device=dev)
        rgb = torch.empty((nq, 3), dtype=torch.uint8, device=dev) if srgb else None
        sl = None if slopes is None else np.ascontiguousarray(slopes, dtype=np.float64)
        ns = 0 if sl is None else sl.shape[0]
        rc = self._L.spoly_render(self._h, mesh_id, chain.encode(), len(chain), endpoints.data_ptr(), width, height,
                                  intensity.data_ptr() if intensity is not None else None, ns,
                                  sl.ctypes.data if sl is not None else None, float(albedo), float(exposure),
                                  rad.data_ptr(), rgb.data_ptr() if rgb is not None else None)
        self._check(rc, "spoly_render")
        return rad.view(height, width), (rgb.view(height, width, 3) if rgb is not None else None)

    def _wrap(self, r: spoly_result, nq: int):
        dev = f"cuda:{self.device}"
        n, m, k = int(r.n_solutions), int(r.n_flagged), int(r.k)
        rep = {f: int(getattr(r.report, f)) for f in REPORT_FIELDS}
        rep.update(ms_cull=r.report.ms_cull, ms_solve=r.report.ms_solve, ms_reduce=r.report.ms_reduce,
                   n_launches=int(r.report.n_launches), n_eval_terms=int(r.report.n_eval_terms),
                   ms_phase1=r.report.ms_phase1, ms_phase2=r.report.ms_phase2, n_rebuilds=int(r.report.n_rebuilds),
                   alg_kflop=int(r.report.alg_kflop), n_jobs_mono=int(r.report.n_jobs_mono),
                   n_jobs_deep=int(r.report.n_jobs_deep), n_elims=int(r.report.n_elims),
                   n_pairs_coarse=int(r.report.n_pairs_coarse), ms_roots=r.report.ms_roots,
                   ms_path=r.report.ms_path, n_refined=int(r.report.n_refined),
                   n_cand_jobs=int(r.report.n_cand_jobs), n_path_jobs=int(r.report.n_path_jobs),
                   n_cull_tests=int(r.report.n_cull_tests), n_truncated=int(r.report.n_truncated),
                   n_big_scan=int(r.report.n_big_scan), n_eval_deep=int(r.report.n_eval_deep),
                   n_rej_visibility=int(r.report.n_rej_visibility))
        return Result(n, m, k, _view(r.query, (n,), "<u4", dev), _view(r.tuple, (n, k), "<u4", dev),
                      _view(r.bary, (n, 2 * k), "<f8", dev), _view(r.contribution, (n,), "<f8", dev),
                      _view(r.residual, (n,), "<f4", dev), _view(r.flags, (n,), "<u4", dev),
                      _view(r.flagged_query, (m,), "<u4", dev), _view(r.flagged_tuple, (m, k), "<u4", dev),
                      _view(r.flagged_flags, (m,), "<u4", dev), _view(r.per_query, (nq,), "<f8", dev), rep)

    def solve(self, chain: str, endpoints, intensity=None, offsets=None, tri_ids=None, mesh_id: int = 0) -> Result:
        """endpoints: CUDA float64 tensor (Q,2,3); intensity: CUDA float64 (Q,) or None;
        offsets/tri_ids: CUDA int32/uint32 CSR tuple list or None (cull pre-pass)."""
        import torch
        assert endpoints.is_cuda and endpoints.dtype == torch.float64 and endpoints.is_contiguous()
        nq = int(endpoints.shape[0])
        tl = None
        if offsets is not None:
            tl = spoly_tuple_list(offsets.data_ptr(), tri_ids.data_ptr())
        r = spoly_result()
        rc = self._L.spoly_solve(self._h, mesh_id, chain.encode(), len(chain), endpoints.data_ptr(), nq,
                                 intensity.data_ptr() if intensity is not None else None,
                                 ctypes.byref(tl) if tl is not None else None, ctypes.byref(r))
        self._check(rc, "spoly_solve")
        self.k = len(chain)
        return self._wrap(r, nq)

    def solve_host(self, chain: str, endpoints: np.ndarray, intensity: np.ndarray = None, mesh_id: int = 0):
        """Host in, host out: returns (per_query numpy (Q,), Result device views)."""
        ep = np.ascontiguousarray(endpoints, dtype=np.float64)
        nq = ep.shape[0]
        it = None if intensity is None else np.ascontiguousarray(intensity, dtype=np.float64)
        pq = np.zeros(nq, np.float64)
        r = spoly_result()
        rc = self._L.spoly_solve_host(self._h, mesh_id, chain.encode(), len(chain), ep.ctypes.data, nq,
                                      it.ctypes.data if it is not None else None, pq.ctypes.data, ctypes.byref(r))
        self._check(rc, "spoly_solve_host")
        return pq, self._wrap(r, nq)

    def last_worklist(self):
        """(pair_query, pair_tuple) of the last solve as int32 torch views (original triangle ids)."""
        pq = ctypes.c_void_p()
        pt = ctypes.c_void_p()
        n = ctypes.c_uint64()
        rc = self._L.spoly_last_worklist(self._h, ctypes.byref(pq), ctypes.byref(pt), ctypes.byref(n))
        self._check(rc, "spoly_last_worklist")
        dev = f"cuda:{self.device}"
        k = self.k or 1
        return _view(pq.value, (n.value,), "<u4", dev), _view(pt.value, (n.value, k), "<u4", dev)

    def bench_fma(self, fp64: bool = True, seconds: float = 1.0) -> float:
        f = ctypes.c_double()
        rc = self._L.spoly_bench_fma(self._h, 1 if fp64 else 0, seconds, ctypes.byref(f))
        self._check(rc, "spoly_bench_fma")
        return f.value
