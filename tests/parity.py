"""GPU-vs-oracle comparison under the parity contract (SURVEY §8(c) "Parity contract").

- counts agree exactly per (query, tuple), except tuples flagged (c14) on EITHER side;
- matched barycentrics agree within `tol_bary` (1e-5 one bounce, 1e-4 two bounces);
- per-query radiance agrees within `tol_rad` relative on queries with no flagged tuple.

Flags may not hide mismatches: each side's flagged fraction (flagged tuples / tuples that side
solved) must stay within `max_flag_frac`; the tuples flagged on one side only (both sides solved
them) must stay within `max_flag_diff` of all flagged tuples (+ `flag_slack` absolute, the
decisions near a threshold that rounding may tip); and at least `min_compared` unflagged chains
must actually be compared.  Set SPOLY_PARITY_LOG=<file> to append every comparison's statistics
(JSON lines).
"""
from __future__ import annotations

import json
import os
from collections import defaultdict

import numpy as np


def _group(query, tuple_, bary):
    d = defaultdict(list)
    for q, t, b in zip(query, tuple_, bary):
        d[(int(q),) + tuple(int(x) for x in np.atleast_1d(t))].append(np.asarray(b, float))
    return d


def _keyset(query, tuple_, k):
    return {(int(q),) + tuple(int(x) for x in t) for q, t in zip(query, np.asarray(tuple_).reshape(-1, k))}


def compare(orc, gpu: dict, nq: int, tol_bary=1e-5, tol_rad=1e-4, max_flag_frac=0.02, min_compared=1,
            max_flag_diff=0.25, flag_slack=2, gpu_pairs=None, orc_pairs=None, gpu_worklist=None, label=""):
    """orc: oracle.Result; gpu: dict of numpy arrays (spoly Result.to_numpy(), optionally "report" and
    "worklist").  gpu_pairs / orc_pairs: tuples each side solved (default: the reports' pair counts).
    gpu_worklist: set of (query, tuple...) keys the GPU solved, used to restrict the one-sided-flag check
    to tuples both sides solved (default: the GPU "worklist" entry when present).  Returns stats dict;
    raises AssertionError with a description on the first violation."""
    k = orc.k
    og = _group(orc.query, orc.tuple, orc.bary)
    gg = _group(gpu["query"], gpu["tuple"].reshape(-1, k), gpu["bary"].reshape(-1, 2 * k))
    flag_o = _keyset(orc.flagged_query, orc.flagged_tuple, k)
    flag_g = _keyset(gpu["flagged_query"], gpu["flagged_tuple"], k)
    flagged = flag_o | flag_g
    flagged_q = {key[0] for key in flagged}
    # --- flags may not hide mismatches: per-side flagged fraction, one-sided flags
    if orc_pairs is None:
        orc_pairs = int(orc.report["pairs_in"])
    if gpu_pairs is None:
        gpu_pairs = int(gpu["report"]["n_pairs_in"]) if "report" in gpu else orc_pairs
    frac_o = len(flag_o) / max(orc_pairs, 1)
    frac_g = len(flag_g) / max(gpu_pairs, 1)
    if gpu_worklist is None and "worklist" in gpu:
        wq, wt = gpu["worklist"]
        gpu_worklist = _keyset(wq, wt, k)
    orc_worklist = _keyset(*orc.worklist, k) if getattr(orc, "worklist", None) is not None else None
    only_g = flag_g - flag_o
    only_o = flag_o - flag_g
    # a tuple only one side's cull kept was never solved by the other: its flag is not a disagreement (the two
    # culls are different sound predicates, SURVEY §8(c) "Cull differences")
    if orc_worklist is not None:
        only_g = {t for t in only_g if t in orc_worklist}
    if gpu_worklist is not None:
        only_o = {t for t in only_o if t in gpu_worklist}
    one_sided = len(only_g) + len(only_o)
    keys = set(og) | set(gg)
    worst = 0.0
    n_cmp = 0
    for key in sorted(keys):
        if key in flagged:
            continue
        a, b = og.get(key, []), gg.get(key, [])
        assert len(a) == len(b), f"{label} count mismatch at (query, tuple)={key}: oracle {a} gpu {b}"
        used = set()
        for x in a:
            d = [np.max(np.abs(x - y)) if j not in used else np.inf for j, y in enumerate(b)]
            j = int(np.argmin(d))
            assert d[j] <= tol_bary, f"{label} vertex mismatch at {key}: oracle {x} gpu {b[j]} (|d|={d[j]:.3g})"
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
    n_rad = 0
    for q in range(nq):
        pairs = [(so[q], sg[q])] + ([] if q in flagged_q else [(orc.per_query[q], gpu["per_query"][q])])
        for ro, rg in pairs:
            rel = abs(ro - rg) / max(abs(ro), 1e-300) if ro != 0 else abs(rg)
            assert rel <= tol_rad, f"{label} radiance mismatch at query {q}: oracle {ro!r} gpu {rg!r} rel {rel:.3g}"
            rad_worst = max(rad_worst, rel)
            n_rad += int(ro != 0)
    st = {"label": label, "compared_solutions": n_cmp, "worst_bary": worst, "worst_rad_rel": rad_worst,
          "compared_radiance": n_rad, "flagged_tuples": len(flagged), "flagged_queries": len(flagged_q),
          "keys": len(keys), "flag_frac_oracle": frac_o, "flag_frac_gpu": frac_g, "flagged_oracle": len(flag_o),
          "flagged_gpu": len(flag_g), "flagged_gpu_only": len(only_g), "flagged_oracle_only": len(only_o),
          "pairs_oracle": orc_pairs, "pairs_gpu": gpu_pairs}
    log = os.environ.get("SPOLY_PARITY_LOG")
    if log:
        with open(log, "a") as f:
            f.write(json.dumps(st, default=float) + "\n")
    assert n_cmp >= min_compared, f"{label} only {n_cmp} unflagged chains compared (< {min_compared}): {st}"
    assert frac_o <= max_flag_frac, f"{label} oracle flagged {frac_o:.3%} of its tuples (> {max_flag_frac:.1%}): {st}"
    assert frac_g <= max_flag_frac, f"{label} GPU flagged {frac_g:.3%} of its tuples (> {max_flag_frac:.1%}): {st}"
    assert one_sided <= flag_slack + max_flag_diff * len(flagged), \
        f"{label} {one_sided} tuples flagged on one side only (of {len(flagged)} flagged): {st}"
    return st
