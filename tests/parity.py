"""GPU-vs-oracle comparison under the parity contract (SURVEY §8(c) "Parity contract").

- counts agree exactly per (query, tuple), except tuples flagged (c14) on EITHER side;
- matched barycentrics agree within `tol_bary` (1e-5 one bounce, 1e-4 two bounces);
- per-query radiance agrees within `tol_rad` relative on queries with no flagged tuple.
"""
from __future__ import annotations

from collections import defaultdict

import numpy as np


def _group(query, tuple_, bary):
    d = defaultdict(list)
    for q, t, b in zip(query, tuple_, bary):
        d[(int(q),) + tuple(int(x) for x in np.atleast_1d(t))].append(np.asarray(b, float))
    return d


def compare(orc, gpu: dict, nq: int, tol_bary=1e-5, tol_rad=1e-4, max_flag_frac=0.02):
    """orc: oracle.Result; gpu: dict of numpy arrays (spoly Result.to_numpy()).  Returns stats dict;
    raises AssertionError with a description on the first violation."""
    k = orc.k
    og = _group(orc.query, orc.tuple, orc.bary)
    gg = _group(gpu["query"], gpu["tuple"].reshape(-1, k), gpu["bary"].reshape(-1, 2 * k))
    flagged = set()
    for q, t in zip(orc.flagged_query, orc.flagged_tuple.reshape(-1, k)):
        flagged.add((int(q),) + tuple(int(x) for x in t))
    for q, t in zip(gpu["flagged_query"], gpu["flagged_tuple"].reshape(-1, k)):
        flagged.add((int(q),) + tuple(int(x) for x in t))
    flagged_q = {key[0] for key in flagged}
    keys = set(og) | set(gg)
    worst = 0.0
    n_cmp = 0
    for key in sorted(keys):
        if key in flagged:
            continue
        a, b = og.get(key, []), gg.get(key, [])
        assert len(a) == len(b), f"count mismatch at (query, tuple)={key}: oracle {a} gpu {b}"
        used = set()
        for x in a:
            d = [np.max(np.abs(x - y)) if j not in used else np.inf for j, y in enumerate(b)]
            j = int(np.argmin(d))
            assert d[j] <= tol_bary, f"vertex mismatch at {key}: oracle {x} gpu {b[j]} (|d|={d[j]:.3g})"
            worst = max(worst, d[j])
            used.add(j)
            n_cmp += 1
    # radiance: per-query sums over the chains of UNFLAGGED tuples (flagged tuples are excluded on both
    # sides, so every query is compared), plus the reported per-query totals on fully unflagged queries
    def unflagged_sum(query, tuple_, contrib):
        s = np.zeros(nq)
        for q, t, c in zip(query, tuple_, contrib):
            if (int(q),) + tuple(int(x) for x in np.atleast_1d(t)) not in flagged:
                s[int(q)] += c
        return s
    so = unflagged_sum(orc.query, orc.tuple, orc.contribution)
    sg = unflagged_sum(gpu["query"], gpu["tuple"].reshape(-1, k), gpu["contribution"])
    rad_worst = 0.0
    for q in range(nq):
        pairs = [(so[q], sg[q])] + ([] if q in flagged_q else [(orc.per_query[q], gpu["per_query"][q])])
        for ro, rg in pairs:
            rel = abs(ro - rg) / max(abs(ro), 1e-300) if ro != 0 else abs(rg)
            assert rel <= tol_rad, f"radiance mismatch at query {q}: oracle {ro!r} gpu {rg!r} rel {rel:.3g}"
            rad_worst = max(rad_worst, rel)
    n_tuples = max(len(keys), 1)
    return {"compared_solutions": n_cmp, "worst_bary": worst, "worst_rad_rel": rad_worst,
            "flagged_tuples": len(flagged), "flagged_queries": len(flagged_q), "keys": len(keys)}
