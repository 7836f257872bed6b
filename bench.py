#!/usr/bin/env python
"""Benchmark of the Specular Polynomials hot path on B200 (driver contract: one JSON line on rank 0).

Workload (BASELINE.json configs[1]): C2 "glints" — 256x256 light samples (queries) x 100,352-triangle
normal-mapped bumpy plane, one-bounce reflection (R), cull pre-pass + fused solve + deterministic
compaction.  One step = one spoly_solve over all 65,536 queries with inputs resident in HBM.

Multi-GPU (torchrun): strong scaling of ONE frame: the frame's query grid is cut into 64 x 64 tiles dealt
round-robin to the ranks; each rank solves its tiles with no collective inside the solve; NCCL
reduces the counters exactly (int64), takes the max (and mean) of the ranks' device times and gathers the per-query
sums back to frame order.

--impl reference: the CPU oracle (plain FP64 C++ transcription of the paper) timed on the host cores on a
bounded sample of the same workload (the reference arm for this tier).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "admissible specular paths/sec and query-tuple solves/sec at 1/2/4/8 B200"
UNIT = "paths/s"

# ---------------------------------------------------------------- algorithmic FLOP model
# Minimal-form FP64 FLOPs of the one-bounce reflection solve (FMA = 2, add/mul/div/sqrt = 1), counted
# from the kernel formulas (DESIGN.md §5 table):
#   phase 1 (k1_phase1: coefficient phase, elimination, Bernstein level, monotone root, pre-check), per pair:
#            decision 75 + setup 18 + a 75 + b 268 + normalise 22 + truncation 10 + coplanarity sign test 16 = 484
#            per pair reaching the elimination (counter n_elims): Bezout 128 + Laplace 316
#                      + normalise r 11 + Bernstein level 155                                = 610
#            + 2 per FMA term of the monotone jobs' Newton evaluations (counter n_eval_terms)
#            + 25 per monotone job with a root (back-substitution: a(., v*) slices + stable quadratic, n_cand_jobs)
#   deep jobs (k1_roots_deep): 2 per FMA term of the derivative recursion (counter n_eval_deep)
#   path (k1_path):
#            + 407 per refined candidate (past the domain pre-check, counter n_refined: one (a,b)
#              Newton step 277, Eq. 3 residual + sides 130)
#            + 250 per admissible chain (analytic ray-differential Jacobian)
#            The path kernel recomputes the coefficient phase from the geometry instead of storing it;
#            that recomputation is implementation overhead, already counted once in phase 1, and is
#            not charged again.
FLOP_PHASE1_PER_PAIR_R = 484
FLOP_PHASE1_PER_ELIM_R = 610
FLOP_PER_EVAL_TERM = 2
FLOP_PER_CANDJOB = 25
FLOP_PER_REFINED_R = 407
FLOP_PER_ADMISSIBLE_R = 250


# one-bounce refraction (T), same accounting: phase 1 per pair: decision 60 + setup 18 + a 75 + b (square
# form, Eq. 9) 656 + normalise/truncate 55 + coplanarity test 16 = 880; per elimination: resultant by
# pseudo-remainder 998 + Bernstein (degree 12) 260 = 1258; refined candidate 730 (b has 28 coefficients);
# admissible 300 (refraction Jacobian).
FLOP_PHASE1_PER_PAIR_T = 880
FLOP_PHASE1_PER_ELIM_T = 1258
FLOP_PER_REFINED_T = 730
FLOP_PER_ADMISSIBLE_T = 300


def flop_model(chain, rep):
    """{kernel: (algorithmic FLOPs per solve, report time key)}.  One bounce: phase 1 (incl. the monotone roots),
    the deep-job kernel and the path kernel; two bounces: the build + scan kernels, whose algorithmic kFLOP the
    kernels count themselves (alg_kflop)."""
    if len(chain) == 1:
        R = chain == "R"
        p1 = (rep["n_pairs_in"] * (FLOP_PHASE1_PER_PAIR_R if R else FLOP_PHASE1_PER_PAIR_T) +
              rep["n_elims"] * (FLOP_PHASE1_PER_ELIM_R if R else FLOP_PHASE1_PER_ELIM_T) +
              rep["n_eval_terms"] * FLOP_PER_EVAL_TERM + rep["n_cand_jobs"] * FLOP_PER_CANDJOB)
        deep = rep["n_eval_deep"] * FLOP_PER_EVAL_TERM
        path = (rep["n_refined"] * (FLOP_PER_REFINED_R if R else FLOP_PER_REFINED_T) +
                rep["n_admissible"] * (FLOP_PER_ADMISSIBLE_R if R else FLOP_PER_ADMISSIBLE_T))
        return {f"k1_phase1<{chain}>": (p1, "ms_phase1"), f"k1_roots_deep<{chain}>": (deep, "ms_roots"),
                f"k1_path<{chain}>": (path, "ms_path")}
    return {f"k2_solve<{chain}>": (rep["alg_kflop"] * 1e3, "ms_phase2")}


# FP64 ALU peak from unit counts and clocks (B200_PROFILING.md: 148 SMs, clocks.max.sm 1965 MHz;
# 64 FP64 FMA lanes per SM per clock)
def fp64_peak(sm_mhz=1965.0, nsm=148):
    return nsm * 64 * 2 * sm_mhz * 1e6


class ClockSampler:
    """SM clock + throttle reasons sampled DURING the timed region: an NVML polling thread (≈2 ms period;
    nvidia-smi's own -lms loop starts too slowly for a 60 ms timed region).  Only samples taken between
    start() and stop() (the first and last timed step) count."""

    REASONS = (("hw_slowdown", 0x8), ("hw_thermal_slowdown", 0x40), ("sw_thermal_slowdown", 0x20),
               ("sw_power_cap", 0x4), ("hw_power_brake_slowdown", 0x80))

    def __init__(self, device_index):
        self.dev = device_index
        self.rows = []  # (t, sm_mhz, max_mhz, reasons bitmask)
        self.t0 = self.t1 = None
        self._stop = False
        self._th = None
        self.h = None
        self.mx = None

    def _handle(self):
        import pynvml
        pynvml.nvmlInit()
        try:
            import torch
            p = torch.cuda.get_device_properties(self.dev)
            bus = "%08X:%02X:%02X.0" % (p.pci_domain_id, p.pci_bus_id, p.pci_device_id)
            return pynvml, pynvml.nvmlDeviceGetHandleByPciBusId(bus)
        except Exception:
            return pynvml, pynvml.nvmlDeviceGetHandleByIndex(self.dev)

    def sample_now(self):
        """One sample from the calling thread (the timed loop calls it after every step's launches, so a
        short timed region has samples even when the polling thread is not scheduled)."""
        if self.h is None:
            return
        nv, h = self.h
        try:
            sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
            rs = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
            self.rows.append((time.perf_counter(), sm, self.mx, rs))
        except Exception:
            pass

    def _run(self):
        while not self._stop:
            self.sample_now()
            time.sleep(0.002)

    def __enter__(self):
        import threading
        try:
            self.h = self._handle()
            self.mx = self.h[0].nvmlDeviceGetMaxClockInfo(self.h[1], self.h[0].NVML_CLOCK_SM)
            self._th = threading.Thread(target=self._run, daemon=True)
            self._th.start()
        except Exception:
            self._th = None
        return self

    def start(self):
        self.t0 = time.perf_counter()

    def stop(self):
        self.t1 = time.perf_counter()

    def __exit__(self, *a):
        self._stop = True
        if self._th is not None:
            self._th.join(timeout=2)

    def summary(self):
        if self.t0 is None:
            return None
        t1 = self.t1 if self.t1 is not None else float("inf")
        rows = [r for r in self.rows if self.t0 <= r[0] <= t1]
        if not rows:
            return None
        reasons = sorted({nm for r in rows for nm, bit in self.REASONS if r[3] & bit})
        return {"sm_mhz": statistics.median(r[1] for r in rows), "sm_max_mhz": max(r[2] for r in rows),
                "reasons": reasons, "samples": len(rows), "source": "nvml: 2 ms polling thread + one sample per timed step, timed region only"}


def oracle_baseline(w, nsample, nthreads=0, worklist=None):
    """The oracle as it stands on a bounded, strided sample of the workload's queries.  worklist (query ids,
    (n, k) tuples of original triangle ids): give the oracle these pairs of the sampled queries as an explicit tuple
    list instead of running its own O(T^2)-per-query two-bounce cull (used at 65,536 triangles, where one query's
    oracle cull alone takes more than 10 minutes)."""
    import oracle
    oracle.build()
    idx = np.linspace(0, w.nqueries - 1, nsample).astype(np.int64)
    sub = w.subset(idx)
    off = ids = None
    what = "oracle cull + solve"
    if worklist is not None:
        wq, wt = worklist
        off = [0]
        ids = []
        for q in idx:
            t = wt[wq == q]
            ids.append(t.reshape(-1))
            off.append(off[-1] + len(t))
        off = np.array(off, np.uint32)
        ids = np.concatenate(ids).astype(np.uint32)
        what = "oracle solve of the GPU cull's work list for those queries"
    t0 = time.perf_counter()
    r = oracle.solve(sub.mesh, w.chain, sub.endpoints, intensity=sub.intensity, offsets=off, tri_ids=ids,
                     nthreads=nthreads)
    dt = time.perf_counter() - t0
    cores = nthreads if nthreads > 0 else (os.cpu_count() or 1)
    return {"value": r.n_solutions / dt, "unit": UNIT, "cores": cores, "kind": "oracle",
            "sample": f"{nsample} of {w.nqueries} queries (strided), full mesh, {what}; "
                      f"{r.n_solutions} paths, {r.report['pairs_in']} pairs in {dt:.2f} s",
            "solves_per_s": r.report["pairs_in"] / dt, "seconds": dt}


def run_reference(args, rank, world):
    """--impl reference: the oracle on the host cores (rank 0 only)."""
    if rank != 0:
        return
    from paper_2405_13409_b200 import workloads as W
    w = W.glints_c2()
    times, paths, pairs = [], 0, 0
    for s in range(args.warmup + args.steps):
        b = oracle_baseline(w, args.ref_sample)
        if s >= args.warmup:
            times.append(b["seconds"])
            paths += b["value"] * b["seconds"]
            pairs += b["solves_per_s"] * b["seconds"]
    tot = sum(times)
    val = paths / tot
    line = {"impl": "reference", "metric": METRIC, "value": val, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "query_tuple_solves_per_s": pairs / tot,
            "config": {"workload": "C2 glints: 65,536 light samples x 100,352-tri bumpy plane, R (sampled "
                                   f"{args.ref_sample} queries per step)", "chain": "R"},
            "cpu_baseline": {"value": val, "unit": UNIT, "cores": os.cpu_count(), "kind": "oracle",
                             "sample": f"{args.ref_sample} strided queries of C2 per step"},
            "e2e": {"value": val, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--res", type=int, default=None, help="query grid side (default: the config's own)")
    ap.add_argument("--config", default="C2", choices=["C1", "C2", "C3", "C4", "C5", "C5RR"],
                    help="workload (BASELINE.json configs; C2 is the driver's bench line)")
    ap.add_argument("--cpu-sample", type=int, default=256)
    ap.add_argument("--ref-sample", type=int, default=256)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--cull-levels", type=int, default=None, help="k=2 cull subdivision levels (default: library)")
    ap.add_argument("--scan-restrict", type=int, default=None, help="k=2 scan restriction (reading R25; default on)")
    ap.add_argument("--k2-tiles", type=int, default=None, help="k=2 cull in query tiles (default on)")
    args = ap.parse_args()

    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))

    if args.impl == "reference":
        run_reference(args, rank, world)
        return

    import torch
    import torch.distributed as dist

    from paper_2405_13409_b200 import spoly
    from paper_2405_13409_b200 import workloads as W

    # one process per GPU; SPOLY_DIST_BACKEND=gloo + more ranks than GPUs is only a functional check of the plumbing
    # (ranks sharing a GPU time-slice it), never a scaling measurement
    local = local % max(torch.cuda.device_count(), 1)
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        backend = os.environ.get("SPOLY_DIST_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)

    scaling = "strong" if world > 1 else "weak"
    shard_idx = None
    kw = {} if args.res is None else {"res": args.res}
    w = W.CONFIGS[args.config](**kw)
    nq_full = w.nqueries
    if world > 1:
        # strong scaling of ONE frame: the frame's res x res query grid in 64 x 64 tiles (halved while
        # there are fewer than 4 tiles per rank), tile t ->
        # rank t mod world; every rank uploads the whole mesh and solves its tiles; no collective inside the solve
        from paper_2405_13409_b200 import dist as D
        side = int(round(nq_full ** 0.5))
        shard_idx = (D.shard_grid_tiles(side, side, world, rank, D.grid_tile_side(side, side, world))
                     if side * side == nq_full
                     else D.shard_tiles(nq_full, world, rank))
        w = w.subset(shard_idx)
    chain = w.chain
    stream = torch.cuda.current_stream(dev)
    kwc = {}
    if args.cull_levels is not None:
        kwc["cull_levels"] = args.cull_levels
    if args.scan_restrict is not None:
        kwc["scan_restrict"] = args.scan_restrict
    if args.k2_tiles is not None:
        kwc["k2_tiles"] = args.k2_tiles
    cfg = spoly.default_config(**kwc)
    ctx = spoly.Context(local, cfg, stream=stream)
    ctx.upload_mesh(w.mesh)
    ep = torch.as_tensor(w.endpoints, dtype=torch.float64, device=dev)
    inten = torch.as_tensor(w.intensity, dtype=torch.float64, device=dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)  # > 126 MB L2

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize(dev)

    for _ in range(max(args.warmup, 3)):
        r = ctx.solve(chain, ep, inten)
    barrier()

    step_ms, solve_ms, reports = [], [], []
    with ClockSampler(local) as clk:
        time.sleep(0.01)  # let the sampler thread take its first sample
        clk.start()
        for s in range(args.steps):
            flush.fill_(s & 0xFF)  # L2 flush between timed iterations (untimed)
            barrier()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            r = ctx.solve(chain, ep, inten)
            e1.record(stream)
            clk.sample_now()
            torch.cuda.synchronize(dev)
            step_ms.append(e0.elapsed_time(e1))
            solve_ms.append(r.report["ms_solve"])
            reports.append(dict(r.report, n_solutions=r.n_solutions))
        clk.stop()
    clocks = clk.summary()
    total_ms = float(sum(step_ms))
    n_paths = sum(x["n_solutions"] for x in reports)
    n_pairs = sum(x["n_pairs_in"] for x in reports)
    launches = sum(x["n_launches"] for x in reports)

    # ---- end to end through the public API with host buffers (H2D endpoints + intensity, D2H per-query)
    e2e = None
    if not args.no_e2e:
        ep_h = np.ascontiguousarray(w.endpoints)
        it_h = np.ascontiguousarray(w.intensity)
        pq, _ = ctx.solve_host(chain, ep_h, it_h)
        e2e_t, e2e_paths = 0.0, 0
        for s in range(args.steps):
            flush.fill_(s & 0xFF)
            barrier()
            t0 = time.perf_counter()
            pq, rr = ctx.solve_host(chain, ep_h, it_h)
            torch.cuda.synchronize(dev)
            e2e_t += time.perf_counter() - t0
            e2e_paths += rr.n_solutions
        e2e = [e2e_paths, e2e_t]

    # ---- cross-rank aggregation (NCCL): exact int64 counter sums, device time max (and mean: imbalance), per-query
    # sums gathered back to frame order
    rank_ms = None
    if world > 1:
        rank_ms = D.allreduce_max_mean(total_ms, dev)
        total_ms = rank_ms[0]
        cnt = D.allreduce_counters({"paths": n_paths, "pairs": n_pairs, "launches": launches,
                                    "e2e_paths": e2e[0] if e2e else 0}, dev)
        n_paths, n_pairs, launches = cnt["paths"], cnt["pairs"], cnt["launches"]
        if e2e:
            e2e = [cnt["e2e_paths"], D.allreduce_max_mean(e2e[1], dev)[0]]
        full_pq = D.gather_per_query(r.per_query.contiguous(), shard_idx, nq_full)
        frame_sum = float(full_pq.sum())

    # ---- roofline of the dominant kernel, from its own launch's CUDA-event time (recorded by the library on
    # the launching stream around each solve kernel, averaged over the timed steps)
    rep = reports[-1]
    peak = fp64_peak()
    phases = {}
    for kname, (flop, key) in flop_model(chain, rep).items():
        tk = statistics.mean(x[key] for x in reports) / 1e3
        phases[kname] = {"ms": tk * 1e3, "flop": flop, "tflops": flop / tk / 1e12 if tk > 0 else None,
                         "frac": flop / tk / peak if tk > 0 else None}
    dname = max(phases, key=lambda kk: phases[kk]["ms"])
    dom = (dname, phases[dname]["flop"], phases[dname]["ms"] / 1e3)
    achieved = dom[1] / dom[2] if dom[2] > 0 else 0.0
    tsum = sum(v["ms"] for v in phases.values()) / 1e3
    phases["solve_total"] = {"ms": tsum * 1e3, "frac": sum(v["flop"] for v in phases.values()) / tsum / peak
                             if tsum > 0 else None}
    traffic = None
    tp = os.path.join(ROOT, "profiles", "solve_traffic.json")
    if os.path.exists(tp):
        try:
            traffic = json.load(open(tp)).get(dom[0], {}).get("dram_bytes_per_launch")
        except Exception:
            traffic = None
    measured_fp64 = ctx.bench_fma(True, 0.5) if rank == 0 else None

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return

    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        wl = None
        if len(chain) == 2 and w.mesh.ntris > 20000:
            lq, lt = ctx.last_worklist()
            wl = (lq.cpu().numpy().view(np.uint32), lt.cpu().numpy().view(np.uint32).reshape(-1, 2))
        cpu = oracle_baseline(w, min(args.cpu_sample, w.nqueries) if len(chain) == 1 else min(4, w.nqueries),
                              worklist=wl)
        cpu.pop("seconds", None)

    line = {
        "metric": METRIC, "value": n_paths / (total_ms / 1e3), "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": max(args.warmup, 3), "ms_per_step": total_ms / args.steps,
        "higher_is_better": True, "scaling": scaling, "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "query_tuple_solves_per_s": n_pairs / (total_ms / 1e3),
        "config": {"workload": ("C2 glints: %d light samples x %d-tri normal-mapped bumpy plane, one-bounce R, "
                                "cull pre-pass + fused FP64 solve + deterministic compaction" % (nq_full, w.mesh.ntris))
                   if args.config == "C2" else "%s %s: %d queries x %d tris, chain %s, cull + solve + compaction" % (
                       args.config, w.name, nq_full, w.mesh.ntris, chain),
                   "queries_per_gpu": w.nqueries, "triangles": w.mesh.ntris, "chain": chain,
                   "queries_total": int(nq_full),
                   "l2": "flushed between timed steps (256 MB write)",
                   "parallelism": ("one frame, query tiles (64x64, halved for small frames) round-robin over %d ranks "
                                   "(strong scaling)" % world
                                   if world > 1 else "single GPU")},
        "paths_per_step_per_gpu": reports[-1]["n_solutions"], "pairs_per_step_per_gpu": reports[-1]["n_pairs_in"],
        "counters": {k: reports[-1][k] for k in ("n_systems", "n_vroots", "n_candidates", "n_admissible", "n_flagged",
                                                 "n_jobs_mono", "n_jobs_deep", "n_eval_terms", "n_rebuilds", "n_elims",
                                                 "n_pairs_coarse", "n_refined", "n_cand_jobs", "n_path_jobs",
                                                 "n_cull_tests", "n_eval_deep", "n_truncated", "n_big_scan")},
        "cull_tests_per_s": reports[-1]["n_cull_tests"] / (statistics.mean(x["ms_cull"] for x in reports) / 1e3)
        if reports[-1]["n_cull_tests"] else None,
        "phase_ms": {"cull": statistics.mean(x["ms_cull"] for x in reports), "solve": statistics.mean(solve_ms),
                     "reduce": statistics.mean(x["ms_reduce"] for x in reports)},
        "roofline": {"bound": "alu", "kernel": dom[0], "achieved": achieved / 1e12, "peak": peak / 1e12,
                     "unit": "TFLOP/s", "frac": achieved / peak, "traffic": traffic, "flop_per_launch": dom[1],
                     "peak_note": "FP64: 148 SMs x 64 FMA/clk x 2 x 1965 MHz (unit counts x clocks.max.sm)",
                     "measured_fp64_fma_tflops": measured_fp64 / 1e12 if measured_fp64 else None,
                     "phases": phases},
        "clocks": clocks,
        "gpu_launches": launches,
    }
    if rank_ms is not None:
        line["ranks"] = {"ms_max": rank_ms[0] / args.steps, "ms_mean": rank_ms[1] / args.steps,
                         "imbalance": rank_ms[0] / rank_ms[1] if rank_ms[1] > 0 else None,
                         "frame_per_query_sum": frame_sum,
                         "note": "per-step device time of the slowest rank (max) and the mean over ranks"}
    if e2e:
        line["e2e"] = {"value": e2e[0] / e2e[1], "unit": UNIT, "h2d_bytes_per_step": int(w.endpoints.nbytes +
                                                                                         w.intensity.nbytes),
                       "d2h_bytes_per_step": int(8 * w.nqueries)}
    if cpu:
        line["cpu_baseline"] = cpu
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
