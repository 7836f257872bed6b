"""Piece-count study ("Impact of the number of pieces"): recall and
time of the two-bounce determinant-sign scan at 10 / 100 / 1000 pieces (PAPER.md:610 uses 100), on the GPU path
and on the oracle, against an independent brute force (tests/bruteforce.py: exact-path camera + light sweeps).

Workloads (seeded, synthetic): planted RR and TT batches (one planted chain per query + 2 decoy pairs) and a C5RR
subset (two facing bumpy mirrors).  Recall = found / (brute-force chains on the same tuples); the oracle and the GPU
must find the same chains at every piece count.  Usage (GPU box): python profiles/piece_study.py [out.json]
"""
from __future__ import annotations

import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import bruteforce  # noqa: E402
import oracle  # noqa: E402
from paper_2405_13409_b200 import workloads as W  # noqa: E402
from planted import planted_many  # noqa: E402

PIECES = (10, 100, 1000)


def planted_batch(chain, n, seed):
    cases = planted_many(seed, chain, n, size=0.15)
    pos, nrm, tri, eps = [], [], [], []
    for i, (m, ids, x0, xk1, bary) in enumerate(cases):
        pos.append(m.pos)
        nrm.append(m.nrm)
        tri.append(m.tri + 6 * i)
        eps.append([x0, xk1])
    mesh = W.Mesh(np.concatenate(pos), np.concatenate(nrm), np.concatenate(tri).astype(np.uint32),
                  cases[0][0].eta_front, cases[0][0].eta_back)
    rng = np.random.default_rng(seed + 1)
    off, ids = [0], []
    for i in range(len(cases)):
        tl = [(2 * i, 2 * i + 1)]
        while len(tl) < 3:
            j, l = rng.integers(0, len(cases), 2)
            if (2 * int(j), 2 * int(l) + 1) not in tl:
                tl.append((2 * int(j), 2 * int(l) + 1))
        for a, b in tl:
            ids += [a, b]
        off.append(off[-1] + len(tl))
    return mesh, np.array(eps, float), np.array(off, np.uint32), np.array(ids, np.uint32)


def truth_set(chain, mesh, ep, off, ids, grid=384):
    """brute-force chains (camera sweep union light sweep) per (query, tuple)"""
    T = {}
    for q in range(len(ep)):
        for t in range(off[q], off[q + 1]):
            tup = (int(ids[2 * t]), int(ids[2 * t + 1]))
            cam = bruteforce.brute_force(chain, mesh, list(tup), ep[q, 0], ep[q, 1], grid=grid,
                                         eta_front=mesh.eta_front, eta_back=mesh.eta_back)
            lit = bruteforce.brute_force_light(chain, mesh, list(tup), ep[q, 0], ep[q, 1], grid=grid,
                                               eta_front=mesh.eta_front, eta_back=mesh.eta_back)
            sols = []
            for c in list(cam) + list(lit):
                if all(np.max(np.abs(np.array(c) - np.array(s))) > 1e-6 for s in sols):
                    sols.append(c)
            T[(q,) + tup] = sols
    return T


def recall(res_query, res_tuple, res_bary, T):
    found = 0
    total = sum(len(v) for v in T.values())
    for key, sols in T.items():
        sel = [i for i in range(len(res_query)) if res_query[i] == key[0] and tuple(res_tuple[i]) == key[1:]]
        for s in sols:
            if any(np.max(np.abs(res_bary[i] - np.array(s))) < 1e-6 for i in sel):
                found += 1
    return found, total


def gpu_solve(mesh, chain, ep, off, ids, pieces):
    import torch
    from paper_2405_13409_b200 import spoly
    ctx = spoly.Context(0, spoly.default_config(pieces=pieces))
    ctx.upload_mesh(mesh)
    e = torch.as_tensor(ep, dtype=torch.float64, device="cuda")
    o = None if off is None else torch.as_tensor(off.astype(np.int32), device="cuda")
    t = None if ids is None else torch.as_tensor(ids.astype(np.int32), device="cuda")
    ctx.solve(chain, e, None, o, t)  # warm-up
    torch.cuda.synchronize()
    r = ctx.solve(chain, e, None, o, t)
    g = r.to_numpy()
    rep = r.report
    ctx.close()
    return g, rep


def main(out):
    use_gpu = True
    try:
        import torch
        use_gpu = torch.cuda.is_available()
    except Exception:
        use_gpu = False
    rows = []
    for chain, n, seed in (("RR", 40, 301), ("TT", 24, 302)):
        mesh, ep, off, ids = planted_batch(chain, n, seed)
        T = truth_set(chain, mesh, ep, off, ids)
        for P in PIECES:
            t0 = time.perf_counter()
            ro = oracle.solve(mesh, chain, ep, offsets=off, tri_ids=ids, cfg=oracle.default_config(pieces=P))
            to = time.perf_counter() - t0
            fo, tot = recall(ro.query, ro.tuple, ro.bary, T)
            row = {"workload": f"planted {chain} ({len(ep)} queries x 3 tuples)", "chain": chain, "pieces": P,
                   "truth_chains": tot, "oracle_found": fo, "oracle_recall": fo / max(tot, 1),
                   "oracle_s": to, "oracle_flagged": int(len(ro.flagged_flags))}
            if use_gpu:
                g, rep = gpu_solve(mesh, chain, ep, off, ids, P)
                fg, _ = recall(g["query"], g["tuple"], g["bary"], T)
                row.update({"gpu_found": fg, "gpu_recall": fg / max(tot, 1), "gpu_solve_ms": rep["ms_solve"],
                            "gpu_flagged": int(len(g["flagged_query"]))})
            rows.append(row)
            print(json.dumps(row), flush=True)
    # C5RR subset: ground truth = brute force on the tuples either side or the 1000-piece scan found a chain in
    w = W.mirrors_rr(res=16, quads=32)
    sub = w.subset(np.arange(0, w.nqueries, 16))
    r1000 = oracle.solve(sub.mesh, "RR", sub.endpoints, cfg=oracle.default_config(pieces=1000))
    wq, wt = r1000.worklist
    keys = sorted({(int(q), int(a), int(b)) for q, (a, b) in zip(r1000.query, r1000.tuple)})
    T = {}
    for k in keys:
        sols = bruteforce.brute_force("RR", sub.mesh, list(k[1:]), sub.endpoints[k[0], 0], sub.endpoints[k[0], 1],
                                      grid=384)
        T[k] = sols
    for P in PIECES:
        t0 = time.perf_counter()
        ro = oracle.solve(sub.mesh, "RR", sub.endpoints, cfg=oracle.default_config(pieces=P))
        to = time.perf_counter() - t0
        fo, tot = recall(ro.query, ro.tuple, ro.bary, T)
        row = {"workload": f"C5RR mirrors subset ({sub.nqueries} receivers, {len(wq)} culled pairs)", "chain": "RR",
               "pieces": P, "truth_chains": tot, "oracle_found": fo, "oracle_recall": fo / max(tot, 1),
               "oracle_s": to, "oracle_solutions": int(ro.n_solutions)}
        if use_gpu:
            g, rep = gpu_solve(sub.mesh, "RR", sub.endpoints, None, None, P)
            fg, _ = recall(g["query"], g["tuple"], g["bary"], T)
            row.update({"gpu_found": fg, "gpu_recall": fg / max(tot, 1), "gpu_solve_ms": rep["ms_solve"],
                        "gpu_solutions": int(len(g["query"]))})
        rows.append(row)
        print(json.dumps(row), flush=True)
    json.dump({"study": "piece count vs recall and time (PAPER.md:789-792)", "rows": rows}, open(out, "w"), indent=1)


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "profiles", "piece_study.json"))
