#!/usr/bin/env python
"""bench.py -- IVF queries/sec on B200 (BASELINE.json metric), one JSON line.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c3] [--impl hivf|reference]

Workload (default `c3`, BASELINE.json configs[2]): 21M x 768 fp32 synthetic
Gaussian mixture, IVF-4096, nprobe=128, k=10, 256-query batches (bench_workload.py).

A step = one batched search (coarse assign -> grouped list scan -> exact top-k)
of one 256-query batch.  `value` = queries/s with queries already in HBM
(hivf_search_device), CUDA events on the library's stream, max over ranks.
`e2e` = the same through the host-buffer C-ABI call hivf_search (pinned host
queries in, results out, copies inside the timed region).  The 64 GB index is
far larger than the 126 MB L2, so no L2 flush is needed between steps.

Multi-GPU (torchrun, one process per GPU): lists are sharded across ranks by
LPT on bytes; each rank searches its shard (exact local top-k), the per-query
candidates are all-gathered with NCCL and merged on device
(hivf_merge_parts_device = merge_topk).  Total index size is fixed as N grows
("scaling": "strong").

`--impl reference` times the reference's own CPU implementation
(oracle/_ref: /root/reference/proj sources compiled unmodified) on the box's
host cores: make_cursor per query + RetrievalEngine::execute(live_math=true),
on a restricted index holding every list probed by a fixed 16-query sample.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "IVF queries/sec (21M×768, nprobe=128, k=10) at 1/2/4/8 B200; % HBM peak"
UNIT = "queries/s"


def log(*a):
    print("[bench]", *a, file=sys.stderr, flush=True)


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.rows = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        try:
            p = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.Q}",
                                  "--format=csv,noheader,nounits", "-lms", "100"],
                                 stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            return
        while not self._stop.is_set():
            line = p.stdout.readline()
            if not line:
                break
            self.rows.append([x.strip() for x in line.split(",")])
        p.terminate()
        try:
            p.wait(timeout=2)
        except Exception:
            p.kill()

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        time.sleep(0.3)
        return self

    def __exit__(self, *exc):
        self._stop.set()
        self._t.join(timeout=3)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for r in self.rows:
            for i, n in enumerate(names):
                if len(r) > 4 + i and r[4 + i].lower() == "active":
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons),
                "samples": len(self.rows)}


# ---------------------------------------------------------------------------
# distributed plumbing (torch.distributed over NCCL; one process per GPU)
# ---------------------------------------------------------------------------

# HIVF_DIST_BACKEND=gloo: functional simulation of the N-rank path on fewer GPUs
# (ranks share devices, collectives staged through host memory).  Never used
# for a reported number; the default and the driver's runs use NCCL.
DIST_BACKEND = os.environ.get("HIVF_DIST_BACKEND", "nccl")


def dist_setup(n_gpus: int):
    import torch
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist
        if DIST_BACKEND == "nccl":
            torch.cuda.set_device(local)
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            local = local % torch.cuda.device_count()
            torch.cuda.set_device(local)
            dist.init_process_group(DIST_BACKEND)
    else:
        torch.cuda.set_device(0)
    return rank, world, local


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def max_over_ranks(x: float, world: int) -> float:
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device="cuda" if DIST_BACKEND == "nccl" else "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def all_gather_parts(out, t):
    """out[world, ...] <- every rank's t (NCCL over NVLink; host-staged for gloo)."""
    import torch.distributed as dist
    if DIST_BACKEND == "nccl":
        dist.all_gather_into_tensor(out, t)
        return
    parts = [p.cpu() for p in out.unbind(0)]
    dist.all_gather(parts, t.cpu())
    for dst, src in zip(out.unbind(0), parts):
        dst.copy_(src)


# ---------------------------------------------------------------------------
# index construction (GPU, chunked, exact same data on every rank)
# ---------------------------------------------------------------------------

def build_shard(wl, ctx, rank, world):
    """Centroids + assignments on GPU, then pack this rank's lists into HBM."""
    import torch
    from bench_workload import list_layout, shard_lists
    from paper_2507_09138_b200 import IvfIndex
    cfg = wl.cfg
    t0 = time.time()
    cents = wl.train_centroids()
    assign = wl.assign_all(cents)
    off, pos, order = list_layout(assign, cfg.k_clusters)
    sizes = (off[1:] - off[:-1]).cpu().numpy()
    owner = shard_lists(sizes, world) if world > 1 else np.zeros(cfg.k_clusters, np.int64)
    own_t = torch.from_numpy(owner == rank).to(wl.device)
    # shard-local CSR: lists not owned by this rank are empty
    my_sizes = torch.where(own_t, off[1:] - off[:-1], torch.zeros_like(off[1:]))
    my_off = torch.zeros_like(off)
    my_off[1:] = torch.cumsum(my_sizes, 0)
    mine_row = own_t[assign]
    # position of each owned row inside the shard CSR
    local_pos = my_off[assign] + (pos - off[assign])
    log(f"rank {rank}: centroids+assign {time.time() - t0:.1f}s; lists {cfg.k_clusters}, "
        f"sizes min {sizes.min()} mean {sizes.mean():.0f} max {sizes.max()}")

    def chunks():
        from bench_workload import CHUNK
        for ci in range(wl.n_chunks()):
            rows = wl.chunk(ci)
            sl = slice(ci * CHUNK, ci * CHUNK + rows.shape[0])
            m = mine_row[sl]
            if world > 1:
                idx = torch.nonzero(m).squeeze(1)
                rows = rows[idx].contiguous()
                p = local_pos[sl][idx].contiguous()
                ids = (idx + ci * CHUNK).contiguous()
            else:
                p = local_pos[sl].contiguous()
                ids = torch.arange(sl.start, sl.stop, device=wl.device, dtype=torch.int64)
            if rows.shape[0]:
                yield p, rows, ids

    t1 = time.time()
    torch.cuda.empty_cache()  # k-means / assignment temporaries -> back to the driver for the lists
    ix = IvfIndex.build_scatter(ctx, cents, my_off.cpu().numpy().astype(np.uint64), 0,
                                int(my_off[-1].item()), chunks())
    log(f"rank {rank}: packed {int(my_off[-1].item())} rows into HBM in {time.time() - t1:.1f}s")
    return ix, cents, sizes, owner, assign, order, off


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------

def run_hivf(args):
    import torch
    from bench_workload import CONFIGS, Workload, algorithmic_bytes, list_bytes
    from paper_2507_09138_b200 import Context
    rank, world, local = dist_setup(args.gpus)
    cfg = CONFIGS[args.config]
    if args.batch:
        cfg.batch = args.batch
    wl = Workload(cfg, device=f"cuda:{local}")
    stream = torch.cuda.current_stream()
    ctx = Context(local, stream)
    # experiment knobs: HIVF_OPTS="tc_qmax=24,seg_rows=8192" (hivf_set_option names)
    for kv in filter(None, os.environ.get("HIVF_OPTS", "").split(",")):
        name, val = kv.split("=")
        ctx.set_option(name.strip(), int(val))
    # --shard R/N: single-GPU measurement of rank R's shard of an N-GPU job (the
    # local search only; the all-gather + merge of the real N-GPU step is not run)
    shard_r, shard_n = (int(x) for x in args.shard.split("/")) if args.shard else (rank, world)
    if args.hbm_budget_gb > 0:  # tiered residency: lists in pinned host memory, hot set in HBM
        ctx.set_option("hbm_list_budget", int(args.hbm_budget_gb * 1e9))
    ix, cents, sizes, owner, assign, order, off = build_shard(wl, ctx, shard_r, shard_n)
    B, npb, k = cfg.batch, cfg.nprobe, cfg.k
    pool = [wl.queries(i) for i in range(args.pool)]
    residency = None
    if args.hbm_budget_gb > 0:
        # the ClusterCacheState target (tiered_cache.cpp:23-36): lists by access
        # frequency over the stream (distinct lists per batch), desc, ties by id
        t0 = time.time()
        freq = np.zeros(cfg.k_clusters, np.int64)
        plan_np = [ix.select_clusters(q.cpu().numpy(), npb) for q in pool]
        for p in plan_np:
            freq[np.unique(p)] += 1
        hot = np.lexsort((np.arange(cfg.k_clusters), -freq)).astype(np.uint32)
        hot = hot[freq[hot] > 0]
        ix.set_residency(hot)
        ix.residency_sync()
        res = ix.residency()
        lb = sizes.astype(np.float64) * ((cfg.dim + 15) // 16 * 16) * 4
        scanned = np.zeros(cfg.k_clusters, bool)
        hit = tot = 0.0
        for p in plan_np:
            u = np.unique(p)
            tot += lb[u].sum()
            hit += lb[u][res[u]].sum()
        residency = {"hbm_list_budget_gb": args.hbm_budget_gb,
                     "index_list_gb": round(float(lb.sum()) / 1e9, 2),
                     "resident_lists": int(res.sum()), "resident_gb": round(float(lb[res].sum()) / 1e9, 2),
                     "scanned_bytes_from_hbm": round(hit / max(tot, 1.0), 4),
                     "policy": "top lists by access frequency over the query stream (freq desc, id asc)",
                     "swap_in_s": round(time.time() - t0, 2)}
        log(f"residency: {residency}")
    # one packed result buffer per rank (ids | dists | counts) so the shard
    # exchange is a single all-gather
    Bk = B * k
    packed = torch.empty(2 * Bk + (B + 1) // 2, dtype=torch.int64, device=wl.device)
    ids = packed[:Bk].view(B, k)
    dd = packed[Bk:2 * Bk].view(torch.float64).view(B, k)
    cnt = packed[2 * Bk:].view(torch.int32)[:B]
    split_assign = world > 1 and B % world == 0
    if world > 1:
        g_packed = torch.empty(world, packed.numel(), dtype=torch.int64, device=wl.device)
        g_ids = torch.empty(world, B, k, dtype=torch.int64, device=wl.device)
        g_d = torch.empty(world, B, k, dtype=torch.float64, device=wl.device)
        g_cnt = torch.empty(world, B, dtype=torch.int32, device=wl.device)
        m_ids, m_d, m_cnt = torch.empty_like(ids), torch.empty_like(dd), torch.empty_like(cnt)
        bs = B // world
        plans_loc = torch.empty(bs, npb, dtype=torch.int32, device=wl.device)
        plans_all = torch.empty(world, bs, npb, dtype=torch.int32, device=wl.device)
    import torch.distributed as dist

    def step(i):
        q = pool[i % len(pool)]
        if world == 1:
            ix.search_device(q, npb, k, ids, dd, cnt)
            return
        if split_assign:
            # coarse assign split across ranks (each assigns B/N queries, the plans
            # are identical to a full assign), plans all-gathered
            ix.assign_device(q[rank * bs:(rank + 1) * bs], npb, plans_loc)
            all_gather_parts(plans_all, plans_loc)
            ix.search_planned_device(q, npb, k, plans_all.view(B, npb), ids, dd, cnt)
        else:
            ix.search_device(q, npb, k, ids, dd, cnt)
        all_gather_parts(g_packed, packed)
        g_ids.copy_(g_packed[:, :Bk].view(world, B, k))
        g_d.copy_(g_packed[:, Bk:2 * Bk].view(torch.float64).view(world, B, k))
        g_cnt.copy_(g_packed[:, 2 * Bk:].view(torch.int32)[:, :B])
        ctx.merge_parts_device(world, B, k, g_ids, g_d, g_cnt, m_ids, m_d, m_cnt)

    for i in range(args.warmup):
        step(i)
    torch.cuda.synchronize()
    st = ctx.stats()
    # our kernels per step: the search call's (stats of the last call) plus, at
    # N>1, the merge and (split assign) the hivf_assign_device kernels
    kernels_per_step = st["kernels_launched"] + (1 if world > 1 else 0) + (4 if split_assign else 0)
    # ---- CUDA graph of the search step (N=1): the library's launch sequence is
    # capturable after a warm call (include/hivf.h); replay removes the launch
    # gaps between the ~15 dependent kernels.  The batch is copied into the
    # captured input buffer each step, so every step still searches new queries.
    graph = None
    # only where launch gaps matter (short steps, e.g. C1/C2); a 10 ms C3 step
    # gains nothing measurable from it and keeps the plain launch path
    t_w0 = time.perf_counter()
    step(0)
    torch.cuda.synchronize()
    short_step = (time.perf_counter() - t_w0) < 2e-3
    if world == 1 and not args.no_graph and short_step:
        try:
            qbuf = torch.empty_like(pool[0])
            qbuf.copy_(pool[0])
            ix.search_device(qbuf, npb, k, ids, dd, cnt)
            torch.cuda.synchronize()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=stream):
                ix.search_device(qbuf, npb, k, ids, dd, cnt)
            torch.cuda.synchronize()
            graph = g
        except Exception as e:  # fall back to direct launches
            log(f"graph capture failed ({e}); timing direct launches")
            graph = None

    def timed_step(i):
        if graph is None:
            step(i)
        else:
            qbuf.copy_(pool[i % len(pool)])
            graph.replay()

    for i in range(args.warmup):
        timed_step(i)
    torch.cuda.synchronize()
    # ---- timed region (value) ----------------------------------------------------
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        barrier(world)
        torch.cuda.synchronize()
        e0.record(stream)
        for i in range(args.steps):
            timed_step(i)
        e1.record(stream)
        torch.cuda.synchronize()
        barrier(world)
    ms = max_over_ranks(e0.elapsed_time(e1), world)
    ms_per_step = ms / args.steps
    value = B * args.steps / (ms / 1e3)
    # ---- per-kernel timing pass (events around each phase, inside the library) ----
    ctx.set_option("time_kernels", 1)
    ctx.set_option("reset_timers", 1)
    tcprof = os.environ.get("HIVF_TCPROF")  # debug: per-CTA stall counters of the scan
    if tcprof:
        ctx.set_option("tc_prof", 1)
    for i in range(args.steps):
        step(i)
    torch.cuda.synchronize()
    if tcprof:
        import ctypes
        from paper_2507_09138_b200 import lib
        n_sm = torch.cuda.get_device_properties(local).multi_processor_count
        buf = np.zeros((n_sm, 16), np.uint64)
        lib().hivf_debug_tc_prof(buf.ctypes.data_as(ctypes.c_void_p), ctypes.c_int(n_sm))
        np.save(tcprof, buf)
        ctx.set_option("tc_prof", 0)
    st = ctx.stats()
    ctx.set_option("time_kernels", 0)
    scan_ms = st["scan_ms"] / max(1, st["timed_calls"])
    assign_ms = st["assign_ms"] / max(1, st["timed_calls"])
    fin_ms = st["finalize_ms"] / max(1, st["timed_calls"])
    # algorithmic bytes of the steps (distinct lists per batch)
    plans = [ix.select_clusters(q.cpu().numpy(), npb) for q in pool]
    my_sizes = np.where(owner == shard_r, sizes, 0)
    lb = [list_bytes(p, my_sizes, cfg.dim) for p in plans]
    ab = [algorithmic_bytes(p, my_sizes, cfg.dim, cfg.k_clusters) for p in plans]
    steps_lb = [lb[i % len(pool)] for i in range(args.steps)]
    steps_ab = [ab[i % len(pool)] for i in range(args.steps)]
    scan_bytes = float(np.mean(steps_lb))
    pp = np.bincount(plans[0].ravel(), minlength=cfg.k_clusters)
    pp = pp[pp > 0]
    probes_per_list = {"mean": round(float(pp.mean()), 2), "p50": int(np.percentile(pp, 50)),
                       "p90": int(np.percentile(pp, 90)), "max": int(pp.max())}
    peak, peak_kind = measured_peaks()
    achieved = scan_bytes / (scan_ms / 1e3) / 1e9
    # DRAM traffic per scan launch from the committed ncu --set full capture of
    # this workload (profiles/ncu_traffic_<config>.json), when one exists
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", f"ncu_traffic_{args.config}.json")) as f:
            tj = json.load(f)
        if world == 1 and not args.shard and not args.hbm_budget_gb:
            traffic = int(tj["dram_bytes_per_launch"])
    except (OSError, KeyError, ValueError):
        pass
    step_gbs = float(np.mean(steps_ab)) / (ms_per_step / 1e3) / 1e9
    # ---- e2e: host buffers through the C-ABI ------------------------------------
    e2e = None
    qh = [torch.empty(B, cfg.dim, dtype=torch.float32, pin_memory=True) for _ in pool]
    for a, b in zip(qh, pool):
        a.copy_(b.cpu())
    if world == 1:
        # the reference-facing C-ABI call with host buffers (hivf_search)
        qn = [a.numpy() for a in qh]
        for i in range(args.warmup):
            ix.search(qn[i % len(qn)], npb, k)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        e0.record(stream)
        for i in range(args.steps):
            ix.search(qn[i % len(qn)], npb, k)
        e1.record(stream)
        torch.cuda.synchronize()
        wall = time.perf_counter() - t0
        e2e_ms = max(e0.elapsed_time(e1), wall * 1e3)
        api = "hivf_search (host buffers, pinned)"
    else:
        # pinned host queries -> HBM, sharded search + all-gather + device merge,
        # merged results -> host, every step inside the timed region
        qd = torch.empty(B, cfg.dim, dtype=torch.float32, device=wl.device)
        h_ids = torch.empty(B, k, dtype=torch.int64, pin_memory=True)
        h_d = torch.empty(B, k, dtype=torch.float64, pin_memory=True)
        h_c = torch.empty(B, dtype=torch.int32, pin_memory=True)

        def e2e_step(i):
            qd.copy_(qh[i % len(qh)], non_blocking=True)
            saved = pool[0]
            pool[0] = qd
            try:
                step(0)
            finally:
                pool[0] = saved
            h_ids.copy_(m_ids, non_blocking=True)
            h_d.copy_(m_d, non_blocking=True)
            h_c.copy_(m_cnt, non_blocking=True)
            torch.cuda.current_stream().synchronize()

        for i in range(args.warmup):
            e2e_step(i)
        barrier(world)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        e0.record(stream)
        for i in range(args.steps):
            e2e_step(i)
        e1.record(stream)
        torch.cuda.synchronize()
        barrier(world)
        wall = time.perf_counter() - t0
        e2e_ms = max_over_ranks(max(e0.elapsed_time(e1), wall * 1e3), world)
        api = ("hivf_assign_device (B/N per rank) + plan all-gather + hivf_search_planned_device"
               " + result all-gather + hivf_merge_parts_device (pinned host in/out)")
    e2e = {"value": B * args.steps / (e2e_ms / 1e3), "unit": UNIT,
           "h2d_bytes_per_step": B * cfg.dim * 4,
           "d2h_bytes_per_step": B * k * (8 + 8) + B * 4, "api": api}
    # ---- CPU baseline + full-scale parity sample (rank 0, N=1) -------------------
    cpu = None
    parity = None
    if world == 1 and rank == 0 and not args.no_cpu:
        cpu, parity = cpu_baseline_and_parity(ix, wl, cents, pool[0], cfg, args)
    if world > 1:
        parity = sharded_parity(ix, wl, cents, pool[0], cfg, step, (m_ids, m_d, m_cnt), rank, world)
    if rank != 0:
        return
    clocks = clk.summary()
    line = {
        "metric": METRIC, "value": round(value, 2), "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_per_step, 4),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32+f64",
        "data": "synthetic gaussian mixture (bench_workload.py), generated on device",
        "launch": "cuda-graph replay of hivf_search_device" if graph is not None else "direct launches",
        "config": {"workload": cfg.describe(), "n_vectors": cfg.n, "dim": cfg.dim,
                   "k_clusters": cfg.k_clusters, "nprobe": npb, "k": k, "batch": B,
                   "query_pool_batches": len(pool),
                   "parallelism": (f"list-sharded x{world}" if not args.shard else
                                   f"one GPU running list shard {shard_r} of {shard_n} (local search "
                                   f"only: value = this shard's queries/s)"),
                   "zipf": cfg.zipf,
                   "probes_per_probed_list": probes_per_list,
                   "l2": "index (%.1f GB) >> 126 MB L2: no flush needed" % (
                       cfg.n * cfg.dim * 4 / 1e9)},
        "e2e": e2e,
        "gpu_launches": kernels_per_step * args.steps,
        "roofline": {"bound": "hbm", "kernel": "k_scan (grouped list scan)",
                     "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                     "frac": round(achieved / peak, 4), "peak_kind": peak_kind,
                     "traffic": traffic,
                     "bytes_per_launch": int(scan_bytes), "launch_ms": round(scan_ms, 4),
                     "step_hbm_frac": round(step_gbs / peak, 4),
                     "phase_ms": {"assign": round(assign_ms, 4), "scan": round(scan_ms, 4),
                                  "finalize": round(fin_ms, 4)}},
        "cpu_baseline": cpu,
        "parity_sample": parity,
        "residency": residency,
        "scan_stats": {"work_items": st["n_work_items"], "fallback_queries": st["n_fallback"],
                       "unique_lists": st["n_unique_lists"]},
        "clocks": clocks,
    }
    print(json.dumps(line), flush=True)


def _ref_restricted_index(rows_by_list, cents, k_clusters):
    """A reference IvfIndex (index_from_assignments, vector_index.cpp:210-235)
    holding only the given lists; select_clusters only reads centroids, so plans
    and results equal the full index's for queries whose plans it covers."""
    import oracle
    corpus = np.concatenate([r for r, _ in rows_by_list.values()]) if rows_by_list else \
        np.zeros((0, cents.shape[1]), np.float32)
    ids = np.concatenate([i for _, i in rows_by_list.values()]) if rows_by_list else \
        np.zeros(0, np.uint64)
    assign = np.concatenate([np.full(len(i), c, np.uint32) for c, (_, i) in rows_by_list.items()]) \
        if rows_by_list else np.zeros(0, np.uint32)
    # index_from_assignments keeps corpus order inside a list: order rows by doc id
    o = np.argsort(ids, kind="stable")
    return oracle.RefIndex.from_assignments(corpus[o], ids[o], cents, assign[o], 0)


def sharded_parity(ix, wl, cents, q0, cfg, step, merged, rank, world, S=4):
    """N>1: every rank runs the reference (oracle/_ref) on its own shard for S
    sample queries (exact local top-k), rank 0 folds the parts with the
    reference's merge_topk and compares with the GPU result of the full
    sharded step (local scan -> all-gather -> device merge)."""
    import torch
    import torch.distributed as dist
    import oracle
    if not oracle.ref_available():
        return None
    Q = q0[:S].cpu().numpy()
    plans = ix.select_clusters(Q, cfg.nprobe)
    sizes = ix.cluster_sizes()
    off = np.zeros(len(sizes) + 1, np.uint64)
    off[1:] = np.cumsum(sizes)
    rows_by_list = {}
    for c in np.unique(plans):
        if sizes[c]:
            rows_by_list[int(c)] = ix.get_rows(int(off[c]), int(sizes[c]))
    ri = _ref_restricted_index(rows_by_list, cents.cpu().numpy(), cfg.k_clusters)
    oi, od, oc = ri.search(Q, cfg.nprobe, cfg.k)
    local = [[(int(oi[b, j]), float(od[b, j])) for j in range(int(oc[b]))] for b in range(S)]
    parts = [None] * world
    dist.all_gather_object(parts, local)
    step(0)  # pool[0] through the sharded GPU path
    torch.cuda.synchronize()
    gi, gd, gc = (t[:S].cpu().numpy() for t in merged)
    exact = True
    for b in range(S):
        ref = []
        for r in range(world):
            ref = oracle.merge_topk(ref, parts[r][b], cfg.k)
        got = [(int(gi[b, j]), float(gd[b, j])) for j in range(int(gc[b]))]
        exact &= [(i, np.float64(d).view(np.uint64)) for i, d in ref] == \
                 [(i, np.float64(d).view(np.uint64)) for i, d in got]
    return {"queries": S, "bit_exact_vs_reference": bool(exact), "nprobe": cfg.nprobe, "k": cfg.k,
            "method": f"reference search per shard ({world} shards) + merge_topk vs GPU "
                      "all-gather + device merge"}


def cpu_baseline_and_parity(ix, wl, cents, q0, cfg, args):
    """Reference CPU path (oracle/_ref) on a bounded sample, timed on this host's
    cores, plus a bit-exact check of our results for the same queries."""
    import oracle
    if not oracle.ref_available():
        try:
            oracle.build()
        except Exception:
            pass
    if not oracle.ref_available():
        return {"value": None, "unit": UNIT, "cores": 0, "kind": "reference",
                "sample": "oracle/_ref not built"}, None
    S = min(args.cpu_sample, q0.shape[0])
    Q = q0[:S].cpu().numpy()
    cents_np = cents.cpu().numpy()
    plans = ix.select_clusters(Q, cfg.nprobe)
    lists = np.unique(plans)
    sizes = ix.cluster_sizes()
    off = np.zeros(len(sizes) + 1, np.uint64)
    off[1:] = np.cumsum(sizes)
    t0 = time.time()
    rows_by_list = {}
    for c in lists:
        r, i = ix.get_rows(int(off[c]), int(sizes[c]))
        rows_by_list[int(c)] = (r, i)
    ri = _ref_restricted_index(rows_by_list, cents_np, cfg.k_clusters)
    log(f"cpu baseline: restricted reference index of {len(lists)} lists "
        f"({sum(len(i) for _, i in rows_by_list.values())} rows) in {time.time() - t0:.1f}s")
    cores = os.cpu_count() or 1
    times = []
    for rep in range(args.cpu_reps):
        ms, oi, od, oc = ri.bench_execute(Q, cfg.nprobe, cfg.k, live=True)
        times.append(ms)
    best = min(times)
    gi, gd, gc = ix.search(Q, cfg.nprobe, cfg.k)
    exact = bool(np.array_equal(gi, oi) and np.array_equal(gd.view(np.uint64), od.view(np.uint64))
                 and np.array_equal(gc, oc))
    cpu = {"value": round(S / (best / 1e3), 3), "unit": UNIT, "cores": cores, "kind": "reference",
           "sample": f"{S} queries of the timed workload (full plans, nprobe={cfg.nprobe}) on a "
                     f"restricted index of the {len(lists)} probed lists; make_cursor xS + "
                     f"RetrievalEngine::execute(live_math=true), best of {len(times)} "
                     f"({', '.join(f'{t / 1e3:.2f}s' for t in times)})"}
    parity = {"queries": S, "bit_exact_vs_reference": exact, "nprobe": cfg.nprobe, "k": cfg.k}
    return cpu, parity


# ---------------------------------------------------------------------------
# reference arm
# ---------------------------------------------------------------------------

def run_c5(args):
    """BASELINE.json configs[4]: heterogeneous node-split retrieval stream,
    p50/p99 latency per concurrency level, both arms on the same batches
    (bench_c5.py).  Single GPU; rank 0 only."""
    import torch
    import oracle
    import bench_c5 as c5
    from bench_workload import CONFIGS, Workload
    from paper_2507_09138_b200 import Context
    if int(os.environ.get("RANK", "0")) != 0:
        return
    cfg = CONFIGS["c2"]  # the stream runs on the C2 index (1M x 768, IVF-1024, nprobe 32)
    torch.cuda.set_device(0)
    wl = Workload(cfg, device="cuda:0")
    ctx = Context(0, torch.cuda.current_stream())  # same stream as the torch-built inputs
    ix, cents, sizes, owner, assign, order, off = build_shard(wl, ctx, 0, 1)
    k = max(cfg.k, c5.K_CACHE)
    Qpool = torch.cat([wl.queries(1000 + i) for i in range(8)]).cpu().numpy()
    budget = int(64 * sizes.mean())  # ~64 lists of rows per sub-stage
    levels = [int(x) for x in os.environ.get("HIVF_C5_LEVELS", "1,8,64,256,512").split(",")]
    ref_ix = None
    if oracle.ref_available() and not args.no_cpu:
        t0 = time.time()
        loff = np.zeros(len(sizes) + 1, np.uint64)
        loff[1:] = np.cumsum(ix.cluster_sizes())
        rows_by_list = {int(c): ix.get_rows(int(loff[c]), int(loff[c + 1] - loff[c]))
                        for c in range(cfg.k_clusters) if loff[c + 1] > loff[c]}
        ref_ix = _ref_restricted_index(rows_by_list, cents.cpu().numpy(), cfg.k_clusters)
        del rows_by_list
        log(f"c5: reference index in {time.time() - t0:.1f}s")
    table = []
    exact_all = True
    for C in levels:
        n_req = max(16, 2 * C)
        # warm pass over the same stream: sizes every scratch / staging buffer
        # (first-call allocations and lazy module loads stay out of the numbers)
        c5.run_stream(c5.GpuArm(ix, cfg.nprobe, k), Qpool, sizes, C, n_req, budget)
        gpu = c5.run_stream(c5.GpuArm(ix, cfg.nprobe, k), Qpool, sizes, C, n_req, budget)
        row = {"concurrency": C, "requests": n_req, "hivf": c5.summarize(gpu)}
        if ref_ix is not None:
            ref = c5.run_stream(c5.RefArm(ref_ix, cfg.nprobe, k), Qpool, sizes, C, n_req, budget)
            row["reference"] = c5.summarize(ref)
            row["bit_exact"] = c5.same_results(gpu, ref)
            exact_all &= row["bit_exact"]
        table.append(row)
        log(f"c5: C={C}: {json.dumps(row)}")
    head = max(table, key=lambda r: r["concurrency"])
    line = {
        "metric": "node-split retrieval stream: p99 stage search latency (configs[4])",
        "value": head["hivf"]["stage_ms"]["p99"], "unit": "ms", "higher_is_better": False,
        "n_gpus": 1, "dtype": "f32+f64",
        "data": "synthetic gaussian mixture (bench_workload.py c2 index), closed-loop "
                "workflow stream (bench_c5.py)",
        "config": {"workload": "C5 node-split stream on 1Mx768 IVF-1024 nprobe=32, "
                               f"heap k={k}, sub-stage budget {budget} rows, "
                               f"concurrency {levels}",
                   "mix": "one-shot 0.4 / HyDE 0.2 / iterative(3 stages) 0.4"},
        "levels": table,
        "parity": {"bit_exact_vs_reference_all_stages": exact_all if ref_ix is not None else None},
        "api": "hivf_select_clusters (make_cursor) + hivf_scan_items per sub-stage, host buffers",
        "reference_arm": "oracle/_ref RetrievalEngine::execute(live_math=true), "
                         f"{os.cpu_count()} host threads" if ref_ix is not None else None,
    }
    print(json.dumps(line), flush=True)


def run_reference(args):
    """The reference's own CPU implementation (oracle/_ref), rank 0 only."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import torch
    import oracle
    from bench_workload import CHUNK, CONFIGS, Workload
    cfg = CONFIGS[args.config]
    if args.batch:
        cfg.batch = args.batch
    if not oracle.ref_available():
        try:
            oracle.build()
        except Exception:
            pass
    if not oracle.ref_available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref (reference sources "
                                                              "compiled) missing"}))
        return
    torch.cuda.set_device(0)
    wl = Workload(cfg)
    t0 = time.time()
    cents = wl.train_centroids()
    assign = wl.assign_all(cents)
    cents_np = cents.cpu().numpy()
    S = min(args.cpu_sample, cfg.batch)
    Q = wl.queries(0)[:S].cpu().numpy()
    # plans from the reference's own select_clusters on a centroid-only index
    empty = oracle.RefIndex.from_assignments(np.zeros((0, cfg.dim), np.float32),
                                             np.zeros(0, np.uint64), cents_np,
                                             np.zeros(0, np.uint32))
    plans = np.stack([empty.select_clusters(q, cfg.nprobe) for q in Q])
    want = torch.zeros(cfg.k_clusters, dtype=torch.bool, device=wl.device)
    want[torch.from_numpy(np.unique(plans).astype(np.int64)).to(wl.device)] = True
    rows, ids, asg = [], [], []
    for ci in range(wl.n_chunks()):
        x = wl.chunk(ci)
        a = assign[ci * CHUNK: ci * CHUNK + x.shape[0]]
        m = torch.nonzero(want[a]).squeeze(1)
        rows.append(x[m].cpu().numpy())
        ids.append((m + ci * CHUNK).cpu().numpy().astype(np.uint64))
        asg.append(a[m].cpu().numpy().astype(np.uint32))
    ri = oracle.RefIndex.from_assignments(np.concatenate(rows), np.concatenate(ids), cents_np,
                                          np.concatenate(asg))
    log(f"reference: restricted index ({int(sum(len(i) for i in ids))} rows) in "
        f"{time.time() - t0:.1f}s")
    for _ in range(args.warmup):
        ri.bench_execute(Q, cfg.nprobe, cfg.k, live=True)
    times = []
    for _ in range(args.steps):
        ms, *_ = ri.bench_execute(Q, cfg.nprobe, cfg.k, live=True)
        times.append(ms)
    tot = sum(times)
    value = S * len(times) / (tot / 1e3)
    cores = os.cpu_count() or 1
    line = {
        "impl": "reference", "metric": METRIC, "value": round(value, 3), "unit": UNIT,
        "n_gpus": int(os.environ.get("WORLD_SIZE", "1")), "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(tot / len(times), 3),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32+f64",
        "data": "synthetic gaussian mixture (bench_workload.py)",
        "config": {"workload": cfg.describe(), "n_vectors": cfg.n, "dim": cfg.dim,
                   "k_clusters": cfg.k_clusters, "nprobe": cfg.nprobe, "k": cfg.k,
                   "batch": cfg.batch, "parallelism": f"{cores} host threads"},
        "cpu_baseline": {"value": round(value, 3), "unit": UNIT, "cores": cores,
                         "kind": "reference",
                         "sample": f"{S} queries per step (full plans) on a restricted index of "
                                   f"the {len(np.unique(plans))} probed lists"},
        "e2e": {"value": round(value, 3), "unit": UNIT, "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c3")
    ap.add_argument("--batch", type=int, default=0)
    ap.add_argument("--impl", default="hivf", choices=["hivf", "reference"])
    ap.add_argument("--pool", type=int, default=8, help="distinct query batches cycled")
    ap.add_argument("--cpu-sample", type=int, default=8)
    ap.add_argument("--cpu-reps", type=int, default=2)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-graph", action="store_true", help="time direct launches instead of a CUDA graph")
    ap.add_argument("--hbm-budget-gb", type=float, default=0.0,
                    help="tiered residency: HBM bytes for list storage (rest in pinned host memory)")
    ap.add_argument("--shard", default="", help="R/N: measure rank R's list shard of an N-GPU job on one GPU")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.config == "c5":
        run_c5(args)
    elif args.impl == "reference":
        run_reference(args)
    else:
        import torch
        local = int(os.environ.get("LOCAL_RANK", "0"))
        if DIST_BACKEND != "nccl":
            local %= torch.cuda.device_count()
        torch.cuda.set_device(local)
        with torch.cuda.stream(torch.cuda.Stream()):  # one explicit stream for torch + hivf
            run_hivf(args)


if __name__ == "__main__":
    main()
