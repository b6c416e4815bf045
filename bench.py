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

Multi-GPU (torchrun, one process per GPU): the library's shard group
(hivf_group_create_nccl): lists sharded by hivf_shard_plan (LPT on bytes, or
on probe frequency x bytes for Zipf streams, hot lists striped), per batch a
slice assign per rank, plan all-gather, exact local search, result
all-gather over NCCL and a device merge_topk.  Total index size and batch are
fixed as N grows ("scaling": "strong").

Parity (`parity_sample`): the GPU outputs of the TIMED steps (one output set
per pool batch) are compared bit-for-bit with the reference on a sample -- the
full batch of two pool batches at C1/C2, 16-query chunks of pool batches 0..3
(64 queries) at C3/C4 -- and the same reference runs are the `cpu_baseline`
(16 queries per chunk = every host thread of the reference's execute works).

`--impl reference` times the reference's own CPU implementation
(oracle/_ref: /root/reference/proj sources compiled unmodified) on the box's
host cores, on the same config and the same query chunks: make_cursor per
query + RetrievalEngine::execute(live_math=true) on a restricted index holding
every list the chunk probes.
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
# shared workload description (identical in both arms -> same_config)
# ---------------------------------------------------------------------------

def config_dict(cfg, args):
    return {"workload": cfg.describe(), "n_vectors": cfg.n, "dim": cfg.dim,
            "k_clusters": cfg.k_clusters, "nprobe": cfg.nprobe, "k": cfg.k, "batch": cfg.batch,
            "zipf": cfg.zipf, "query_pool_batches": args.pool,
            "seeds": {"corpus": 1, "queries": 2},
            "index": "train_centroids (Lloyd on a 48K-row sample) + compute_assignments over every row",
            "l2": "index (%.1f GB) >> 126 MB L2: no flush needed" % (cfg.n * cfg.dim * 4 / 1e9)}


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def sample_plan(cfg, args):
    """The queries the reference is timed / compared on: the full batch of pool
    batches 0..1 when the whole index is small (C1/C2); otherwise 16 queries
    (= host threads, so every core of the reference's execute works) from each
    of pool batches 0..3, at a different row offset in every batch (C3/C4):
    64 queries.  Returns [(pool batch, first row, n rows)]."""
    small = cfg.n * cfg.dim * 4 <= 8e9
    if small:
        return [(j, 0, cfg.batch) for j in range(min(2, args.pool))]
    S = max(1, min(args.cpu_sample, cfg.batch))
    out = []
    for j in range(min(4, args.pool)):
        first = (j * (cfg.batch // 4)) % max(1, cfg.batch - S + 1)
        out.append((j, first, S))
    return out


# ---------------------------------------------------------------------------
# index construction (GPU, chunked; the same data on every rank)
# ---------------------------------------------------------------------------

def list_weights(ix_cents_only, wl, cfg, n_batches=8, group=64):
    """Expected scan passes per batch of every list (its probe frequency) from
    a warm-up sample of the query stream (batches disjoint from the timed
    pool): mean over batches of ceil(probes / group) -- the ClusterCacheState
    frequency counter (tiered_cache.cpp:10-14) in bytes-streamed units."""
    K = cfg.k_clusters
    acc = np.zeros(K)
    for i in range(n_batches):
        p = ix_cents_only.select_clusters(wl.queries(100_000 + i).cpu().numpy(), cfg.nprobe)
        cnt = np.bincount(p.ravel(), minlength=K)
        acc += np.ceil(cnt / group)
    w = acc / n_batches
    return np.maximum(w, 0.5 / n_batches)  # never-seen lists still balance by size


def build_index(wl, ctx, rank, world, cents=None, assign=None):
    """Centroids (synthetic input) + library compute_assignments, shard plan
    (hivf_shard_plan: frequency-weighted LPT + striped hot lists), and this
    rank's lists packed into HBM (hivf_index_begin / add_rows_at / finish)."""
    import torch
    from bench_workload import CHUNK, list_layout
    from paper_2507_09138_b200 import IvfIndex, shard_local_lists, shard_plan
    cfg = wl.cfg
    info = {}
    t0 = time.time()
    if cents is None:
        cents = wl.train_centroids()
    torch.cuda.synchronize()
    info["centroids_s"] = round(time.time() - t0, 2)
    t1 = time.time()
    if assign is None:
        assign = wl.library_assign(ctx, cents)
    torch.cuda.synchronize()
    info["compute_assignments_s"] = round(time.time() - t1, 2)
    info["compute_assignments"] = "hivf_compute_assignments (libhivf), every row"
    off, pos, order = list_layout(assign, cfg.k_clusters)
    sizes = (off[1:] - off[:-1]).cpu().numpy().astype(np.uint64)
    weights = None
    if world > 1 and cfg.zipf > 0:
        probe = IvfIndex.build_scatter(ctx, cents, np.zeros(cfg.k_clusters + 1, np.uint64), 0, 0, iter(()))
        weights = list_weights(probe, wl, cfg)
        probe.close()
    owner = shard_plan(sizes, world, weights=weights) if world > 1 else np.zeros(cfg.k_clusters, np.uint32)
    off_np = off.cpu().numpy().astype(np.uint64)
    loc_off, src_first = shard_local_lists(off_np, owner, world, rank)
    lo_t = torch.from_numpy((src_first - off_np[:-1]).astype(np.int64)).to(wl.device)
    nl_t = torch.from_numpy((loc_off[1:] - loc_off[:-1]).astype(np.int64)).to(wl.device)
    lof_t = torch.from_numpy(loc_off[:-1].astype(np.int64)).to(wl.device)
    rank_in_list = pos - off[assign]
    rel = rank_in_list - lo_t[assign]
    mine_row = (rel >= 0) & (rel < nl_t[assign])
    local_pos = lof_t[assign] + rel
    info["shard"] = {"ranks": world, "striped_lists": int((owner == 0xFFFFFFFF).sum()),
                     "weights": "probe frequency (warm-up batches)" if weights is not None else "bytes"}
    log(f"rank {rank}: centroids {info['centroids_s']}s, compute_assignments {info['compute_assignments_s']}s; "
        f"lists {cfg.k_clusters}, sizes min {sizes.min()} mean {sizes.mean():.0f} max {sizes.max()}")

    def chunks():
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

    t2 = time.time()
    torch.cuda.empty_cache()
    n_loc = int(loc_off[-1])
    ix = IvfIndex.build_scatter(ctx, cents, loc_off, 0, n_loc, chunks())
    info["pack_s"] = round(time.time() - t2, 2)
    info["local_rows"] = n_loc
    log(f"rank {rank}: packed {n_loc} rows into HBM in {info['pack_s']}s")
    local_sizes = (loc_off[1:] - loc_off[:-1]).astype(np.uint64)
    return ix, cents, sizes, local_sizes, owner, assign, info


def make_group(ix, rank, world):
    """The library's shard group for this rank: NCCL (one process per GPU), or
    the host all-gather transport for the HIVF_DIST_BACKEND=gloo simulation."""
    import torch
    import torch.distributed as dist
    from paper_2507_09138_b200 import ShardGroup, nccl_unique_id
    if DIST_BACKEND == "nccl":
        obj = [nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        return ShardGroup.nccl(ix, world, rank, obj[0])

    def allgather(send: bytes) -> bytes:
        t = torch.frombuffer(bytearray(send), dtype=torch.uint8)
        out = [torch.empty_like(t) for _ in range(world)]
        dist.all_gather(out, t)
        return b"".join(bytes(o.numpy()) for o in out)
    return ShardGroup.host_allgather(ix, world, rank, allgather)


# ---------------------------------------------------------------------------
# reference CPU path on a sample (parity + cpu_baseline)
# ---------------------------------------------------------------------------

def restricted_ref_index(ix, cents_np, lists, local_sizes):
    """The reference's IvfIndex holding only `lists` (their rows read back from
    HBM in list order, i.e. index_from_assignments order); select_clusters only
    reads centroids, so searches whose plans these lists cover equal the full
    index's (ref_index_from_csr, oracle/ref_shim.cpp)."""
    import oracle
    K = cents_np.shape[0]
    dim = cents_np.shape[1]
    off = np.zeros(K + 1, np.uint64)
    sz = np.zeros(K, np.uint64)
    sz[lists] = local_sizes[lists]
    off[1:] = np.cumsum(sz)
    gl_off = np.zeros(K + 1, np.uint64)
    gl_off[1:] = np.cumsum(local_sizes)
    T = int(off[-1])
    vec = np.empty((T, dim), np.float32)
    ids = np.empty(T, np.uint64)
    for c in lists:
        n = int(sz[c])
        if n:
            ix.get_rows_into(int(gl_off[c]), n, vec[int(off[c]):int(off[c]) + n], ids[int(off[c]):int(off[c]) + n])
    ri = oracle.RefIndex.from_csr(cents_np, off, vec, ids)
    del vec, ids
    return ri, T


def reference_on_sample(ix, cents, cfg, args, pool_np, local_sizes, outs=None, time_it=True):
    """For every sample chunk: restricted reference index, the reference's
    make_cursor x S + RetrievalEngine::execute(live_math=true) (timed), and a
    bit-exact comparison with the rows of the TIMED batch's GPU outputs."""
    import oracle
    cents_np = cents.cpu().numpy()
    nproc = os.cpu_count() or 1
    tot_ms = 0.0
    tot_q = 0
    exact = True
    mism = 0
    parts = []
    rows_total = 0
    results = []
    for (j, first, S) in sample_plan(cfg, args):
        Q = pool_np[j][first:first + S]
        plans = ix.select_clusters(Q, cfg.nprobe)
        lists = np.unique(plans)
        t0 = time.time()
        ri, T = restricted_ref_index(ix, cents_np, lists, local_sizes)
        t_build = time.time() - t0
        ms, oi, od, oc = ri.bench_execute(Q, cfg.nprobe, cfg.k, live=True)
        del ri
        tot_ms += ms
        tot_q += S
        rows_total += T
        results.append((j, first, S, oi, od, oc))
        if outs is not None:
            gi, gd, gc = (t[first:first + S] for t in outs[j])
            ok = (np.array_equal(gc, oc) and np.array_equal(gi, oi)
                  and np.array_equal(gd.view(np.uint64), od.view(np.uint64)))
            exact &= ok
            mism += int((~(gi == oi).all(1)).sum() + (gc != oc).sum())
        parts.append({"pool_batch": j, "rows": [first, first + S], "lists": int(len(lists)),
                      "index_rows": T, "execute_ms": round(ms, 1), "index_build_s": round(t_build, 1)})
        log(f"reference sample: batch {j} rows {first}:{first + S}: {len(lists)} lists, {T} rows, "
            f"execute {ms / 1e3:.2f}s (index {t_build:.1f}s)")
    info = {"queries": tot_q, "chunks": parts, "ms": tot_ms,
            "threads_used": min(max(S for _, _, S in sample_plan(cfg, args)), nproc), "nproc": nproc,
            "cpu_model": cpu_model()}
    parity = None
    if outs is not None:
        parity = {"queries": tot_q, "batch": cfg.batch, "from_timed_batch": True,
                  "pool_batches": sorted({j for j, _, _ in sample_plan(cfg, args)}),
                  "bit_exact": bool(exact), "mismatched_queries": mism,
                  "nprobe": cfg.nprobe, "k": cfg.k,
                  "method": "GPU outputs of the timed steps vs the reference (oracle/_ref) make_cursor + "
                            "RetrievalEngine::execute on a restricted index of the probed lists"}
    return info, parity, results


def cpu_baseline_line(info, cfg):
    return {"value": round(info["queries"] / (info["ms"] / 1e3), 3), "unit": UNIT,
            "cores": info["threads_used"], "threads_used": info["threads_used"], "nproc": info["nproc"],
            "cpu_model": info["cpu_model"], "kind": "reference",
            "sample": f"{info['queries']} queries of the timed workload in {len(info['chunks'])} chunks "
                      f"({', '.join(str(c['pool_batch']) + ':' + str(c['rows'][0]) + '-' + str(c['rows'][1]) for c in info['chunks'])}"
                      f"; full plans, nprobe={cfg.nprobe}, k={cfg.k}); per chunk make_cursor x S + "
                      f"RetrievalEngine::execute(live_math=true) over a restricted index of the probed lists"}


def sharded_parity(ix, cents, cfg, args, pool_np, local_sizes, outs, rank, world):
    """N>1: every rank runs the reference on its own shard for the sample
    queries (exact local top-k), rank 0 folds the parts with the reference's
    merge_topk and compares with the merged GPU outputs of the timed steps."""
    import torch.distributed as dist
    import oracle
    if not oracle.ref_available():
        return None
    _, _, res = reference_on_sample(ix, cents, cfg, args, pool_np, local_sizes, None)
    local = [[[(int(oi[b, e]), float(od[b, e])) for e in range(int(oc[b]))] for b in range(S)]
             for (_, _, S, oi, od, oc) in res]
    parts = [None] * world
    dist.all_gather_object(parts, local)
    if rank != 0:
        return None
    exact = True
    nq = 0
    for ci, (j, first, S, _, _, _) in enumerate(res):
        gi, gd, gc = (t[first:first + S] for t in outs[j])
        for b in range(S):
            ref = []
            for r in range(world):
                ref = oracle.merge_topk(ref, parts[r][ci][b], cfg.k)
            got = [(int(gi[b, e]), float(gd[b, e])) for e in range(int(gc[b]))]
            exact &= [(i, np.float64(d).view(np.uint64)) for i, d in ref] == \
                     [(i, np.float64(d).view(np.uint64)) for i, d in got]
            nq += 1
    return {"queries": nq, "batch": cfg.batch, "from_timed_batch": True, "bit_exact": bool(exact),
            "nprobe": cfg.nprobe, "k": cfg.k,
            "method": f"reference search per shard ({world} shards) + merge_topk vs the merged GPU "
                      "outputs of the timed steps (hivf_group_search_device)"}


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
    if args.shard:
        return run_shard_sweep(args, wl, ctx, cfg)
    if args.hbm_budget_gb > 0:  # tiered residency: lists in pinned host memory, hot set in HBM
        ctx.set_option("hbm_list_budget", int(args.hbm_budget_gb * 1e9))
    ix, cents, sizes, local_sizes, owner, assign, build_info = build_index(wl, ctx, rank, world)
    del assign
    B, npb, k = cfg.batch, cfg.nprobe, cfg.k
    pool = [wl.queries(i) for i in range(args.pool)]
    pool_np = [q.cpu().numpy() for q in pool]
    residency = setup_residency(ix, cfg, args, pool_np, sizes) if args.hbm_budget_gb > 0 else None
    group = make_group(ix, rank, world) if world > 1 else None
    # one output set per pool batch: the timed steps' results stay for parity
    outs_t = [(torch.zeros(B, k, dtype=torch.int64, device=wl.device),
               torch.zeros(B, k, dtype=torch.float64, device=wl.device),
               torch.zeros(B, dtype=torch.int32, device=wl.device)) for _ in pool]

    def step(i):
        j = i % len(pool)
        o = outs_t[j]
        if group is None:
            ix.search_device(pool[j], npb, k, *o)
        else:
            group.search_device(pool[j], npb, k, *o)

    for i in range(args.warmup):
        step(i)
    torch.cuda.synchronize()
    barrier(world)
    kernels_per_step = ctx.stats()["kernels_launched"]
    # ---- CUDA graphs of the search step (N=1, short steps only): the library's
    # launch sequence is capturable after a warm call (include/hivf.h); one
    # graph per pool batch (its own input and outputs), so every replay
    # searches a different batch with no extra copies
    graphs = None
    t_w0 = time.perf_counter()
    step(0)
    torch.cuda.synchronize()
    short_step = (time.perf_counter() - t_w0) < 2e-3
    if world == 1 and not args.no_graph and short_step:
        try:
            graphs = []
            for j in range(len(pool)):
                step(j)
                torch.cuda.synchronize()
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g, stream=stream):
                    step(j)
                graphs.append(g)
            torch.cuda.synchronize()
        except Exception as e:  # fall back to direct launches
            log(f"graph capture failed ({e}); timing direct launches")
            graphs = None

    def timed_step(i):
        if graphs is None:
            step(i)
        else:
            graphs[i % len(pool)].replay()

    for i in range(args.warmup):
        timed_step(i)
    torch.cuda.synchronize()
    # ---- timed region (value) ----------------------------------------------------
    # HIVF_NCU_RANGE=1: the profiler range is the timed region only (ncu
    # --profile-from-start off), so launch lists skip the index build
    ncu_range = bool(os.environ.get("HIVF_NCU_RANGE"))
    if ncu_range:
        torch.cuda.cudart().cudaProfilerStart()
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
    if ncu_range:
        torch.cuda.cudart().cudaProfilerStop()
    ms = max_over_ranks(e0.elapsed_time(e1), world)
    ms_per_step = ms / args.steps
    value = B * args.steps / (ms / 1e3)
    outs = [tuple(t.cpu().numpy() for t in o) for o in outs_t]
    outs = [(a.view(np.uint64), b, c.view(np.uint32)) for a, b, c in outs]
    # ---- optional scan stall counters (HIVF_TCPROF=<out.npy>; profiles/tcprof.py) ----
    if os.environ.get("HIVF_TCPROF"):
        from paper_2507_09138_b200 import lib
        ctx.set_option("tc_prof", 1)
        for i in range(args.steps):
            step(i)
        torch.cuda.synchronize()
        prof = np.zeros((ctx.device_info()["sm_count"], 16), np.uint64)
        lib().hivf_debug_tc_prof(prof.ctypes.data, prof.shape[0])
        ctx.set_option("tc_prof", 0)
        np.save(os.environ["HIVF_TCPROF"], prof)
        log(f"scan stall counters over {args.steps} steps -> {os.environ['HIVF_TCPROF']}")
    # ---- per-kernel timing pass (events around each phase, inside the library) ----
    ctx.set_option("time_kernels", 1)
    ctx.set_option("reset_timers", 1)
    for i in range(args.steps):
        step(i)
    torch.cuda.synchronize()
    st = ctx.stats()
    ctx.set_option("time_kernels", 0)
    scan_ms = st["scan_ms"] / max(1, st["timed_calls"])
    assign_ms = st["assign_ms"] / max(1, st["timed_calls"])
    fin_ms = st["finalize_ms"] / max(1, st["timed_calls"])
    # algorithmic bytes of the steps (distinct lists per batch) over
    # this rank's rows
    plans = [ix.select_clusters(q, npb) for q in pool_np]
    elem = st["scan_filter_bits"] // 8  # 2: the scan streamed the fp16 filter copy
    lb = [list_bytes(p, local_sizes, cfg.dim, elem) for p in plans]
    ab = [algorithmic_bytes(p, local_sizes, cfg.dim, cfg.k_clusters, elem) for p in plans]
    scan_bytes = float(np.mean([lb[i % len(pool)] for i in range(args.steps)]))
    step_ab = float(np.mean([ab[i % len(pool)] for i in range(args.steps)]))
    pp = np.bincount(plans[0].ravel(), minlength=cfg.k_clusters)
    pp = pp[pp > 0]
    probes_per_list = {"mean": round(float(pp.mean()), 2), "p50": int(np.percentile(pp, 50)),
                       "p90": int(np.percentile(pp, 90)), "max": int(pp.max())}
    peak, peak_kind = measured_peaks()
    achieved = scan_bytes / (scan_ms / 1e3) / 1e9
    scan_ms_all = [max_over_ranks(scan_ms, world)] if world > 1 else [scan_ms]
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", f"ncu_traffic_{args.config}"
                               f"{'_b%d' % B if B != 256 else ''}{'_h16' if elem == 2 else ''}.json")) as f:
            tj = json.load(f)
        if world == 1 and not args.hbm_budget_gb:
            traffic = int(tj["dram_bytes_per_launch"])
    except (OSError, KeyError, ValueError):
        pass
    # ---- e2e: host buffers through the public C-ABI ------------------------------
    # the step's queries come from pinned host memory (page-locked once, outside
    # the timed region), so the H2D copy inside hivf_search is a direct DMA
    qh = [torch.from_numpy(np.ascontiguousarray(q)).pin_memory().numpy() for q in pool_np]
    for i in range(args.warmup):
        (ix.search(qh[i % len(qh)], npb, k) if group is None else group.search(qh[i % len(qh)], npb, k))
    torch.cuda.synchronize()
    barrier(world)
    t0 = time.perf_counter()
    e0.record(stream)
    for i in range(args.steps):
        (ix.search(qh[i % len(qh)], npb, k) if group is None else group.search(qh[i % len(qh)], npb, k))
    e1.record(stream)
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    barrier(world)
    e2e_ms = max_over_ranks(max(e0.elapsed_time(e1), wall * 1e3), world)
    api = "hivf_search (host buffers)" if group is None else \
        "hivf_group_search (host buffers; NCCL shard group: slice assign, plan all-gather, local search, " \
        "result all-gather, device merge_topk)"
    e2e = {"value": round(B * args.steps / (e2e_ms / 1e3), 2), "unit": UNIT,
           "h2d_bytes_per_step": B * cfg.dim * 4, "d2h_bytes_per_step": B * k * (8 + 8) + B * 4, "api": api, "host_queries": "pinned"}
    # ---- CPU baseline + parity of the timed batches --------------------------------
    cpu = parity = None
    if not args.no_cpu:
        import oracle
        if not oracle.ref_available():
            try:
                oracle.build()
            except Exception:
                pass
        if world == 1 and oracle.ref_available():
            info, parity, _ = reference_on_sample(ix, cents, cfg, args, pool_np, local_sizes, outs)
            cpu = cpu_baseline_line(info, cfg)
        elif world > 1:
            parity = sharded_parity(ix, cents, cfg, args, pool_np, local_sizes, outs, rank, world)
    if residency is not None:
        # the scan's bytes: the fp16 filter copy of every list lives in HBM
        # (outside the budget), so the scan never crosses PCIe; the budget
        # governs where the exact re-rank reads the fp32 rows
        residency["scan_reads"] = ("fp16 filter copy, every list in HBM" if elem == 2
                                   else "fp32 lists: resident from the HBM pool, cold over PCIe")
        if elem == 2:
            residency["exact_rows_from_hbm"] = residency.pop("scanned_bytes_from_hbm")
    if rank != 0:
        return
    clocks = clk.summary()
    line = {
        "metric": METRIC, "value": round(value, 2), "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_per_step, 4),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        # filter: fp16 filter copy x fp16 queries, fp32 accumulate (or tf32 over the
        # fp32 lists); results: the reference's exact fp64 distances
        "dtype": "f16+f32+f64" if elem == 2 else "f32+f64",
        "filter": "fp16 filter copy (DESIGN.md 3a), exact fp64 re-rank" if elem == 2 else "fp32 lists (tf32), exact fp64 re-rank",
        "data": "synthetic gaussian mixture (bench_workload.py), generated on device",
        "launch": "cuda-graph replay of hivf_search_device" if graphs is not None else "direct launches",
        "api": "hivf_search_device" if group is None else "hivf_group_search_device (NCCL shard group)",
        "config": config_dict(cfg, args),
        "parallelism": f"lists sharded over {world} GPUs" if world > 1 else "one GPU, whole index",
        "e2e": e2e,
        "gpu_launches": kernels_per_step * args.steps,
        "roofline": {"bound": "hbm", "kernel": "k_scan_tc (grouped list scan)",
                     "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                     "frac": round(achieved / peak, 4), "peak_kind": peak_kind,
                     "traffic": traffic,
                     "bytes_per_launch": int(scan_bytes), "launch_ms": round(scan_ms, 4),
                     "bytes_basis": ("distinct probed rows x dim x 2 B (the fp16 filter copy the scan streams)"
                                     if elem == 2 else "distinct probed rows x dim x 4 B (fp32 lists)"),
                     "launch_ms_max_over_ranks": round(scan_ms_all[0], 4),
                     "step_hbm_frac": round(step_ab / (ms_per_step / 1e3) / 1e9 / peak, 4),
                     "phase_ms": {"assign": round(assign_ms, 4), "scan": round(scan_ms, 4),
                                  "finalize": round(fin_ms, 4)},
                     "probes_per_probed_list": probes_per_list},
        "cpu_baseline": cpu,
        "parity_sample": parity,
        "index_build": build_info,
        "residency": residency,
        "scan_stats": {"work_items": st["n_work_items"], "fallback_queries": st["n_fallback"],
                       "unique_lists": st["n_unique_lists"]},
        "clocks": clocks,
    }
    print(json.dumps(line), flush=True)


def setup_residency(ix, cfg, args, pool_np, sizes):
    """Tiered residency: the ClusterCacheState target (tiered_cache.cpp:23-36)
    -- lists by access frequency over the stream (distinct lists per batch),
    desc, ties by id -- made resident in the HBM pool."""
    t0 = time.time()
    freq = np.zeros(cfg.k_clusters, np.int64)
    plan_np = [ix.select_clusters(q, cfg.nprobe) for q in pool_np]
    for p in plan_np:
        freq[np.unique(p)] += 1
    hot = np.lexsort((np.arange(cfg.k_clusters), -freq)).astype(np.uint32)
    hot = hot[freq[hot] > 0]
    ix.set_residency(hot)
    ix.residency_sync()
    res = ix.residency()
    lb = sizes.astype(np.float64) * ((cfg.dim + 15) // 16 * 16) * 4
    hit = tot = 0.0
    for p in plan_np:
        u = np.unique(p)
        tot += lb[u].sum()
        hit += lb[u][res[u]].sum()
    out = {"hbm_list_budget_gb": args.hbm_budget_gb, "index_list_gb": round(float(lb.sum()) / 1e9, 2),
           "resident_lists": int(res.sum()), "resident_gb": round(float(lb[res].sum()) / 1e9, 2),
           "scanned_bytes_from_hbm": round(hit / max(tot, 1.0), 4),
           "policy": "top lists by access frequency over the query stream (freq desc, id asc)",
           "swap_in_s": round(time.time() - t0, 2)}
    log(f"residency: {out}")
    return out


def run_shard_sweep(args, wl, ctx, cfg):
    """--shard R/N or all/N: on ONE GPU, build and time rank R's (or every
    rank's, one after another) list shard of an N-GPU job -- the local search
    of the sharded step (slice assign, the all-gathers and the merge are not
    run).  Grounds the N-GPU projection in every shard's step time."""
    import torch
    r_s, n_s = args.shard.split("/")
    N = int(n_s)
    ranks = list(range(N)) if r_s == "all" else [int(r_s)]
    cents = wl.train_centroids()
    t0 = time.time()
    assign = wl.library_assign(ctx, cents)
    t_assign = time.time() - t0
    B, npb, k = cfg.batch, cfg.nprobe, cfg.k
    pool = [wl.queries(i) for i in range(args.pool)]
    pool_np = [q.cpu().numpy() for q in pool]
    rows = []
    # one output set per pool batch: the timed steps' results stay for parity
    outs_t = [(torch.zeros(B, k, dtype=torch.int64, device=wl.device),
               torch.zeros(B, k, dtype=torch.float64, device=wl.device),
               torch.zeros(B, dtype=torch.int32, device=wl.device)) for _ in pool]
    o = outs_t[0]
    stream = torch.cuda.current_stream()
    for r in ranks:
        ix, _, sizes, local_sizes, owner, _, info = build_index(wl, ctx, r, N, cents, assign)
        for i in range(args.warmup):
            ix.search_device(pool[i % len(pool)], npb, k, *outs_t[i % len(pool)])
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for i in range(args.steps):
            ix.search_device(pool[i % len(pool)], npb, k, *outs_t[i % len(pool)])
        e1.record(stream)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / args.steps
        parity = None
        if not args.no_cpu:  # this shard's exact local top-k vs the reference on the shard's lists
            outs = [tuple(t.cpu().numpy() for t in ot) for ot in outs_t]
            outs = [(a.view(np.uint64), b, c.view(np.uint32)) for a, b, c in outs]
            _, parity, _ = reference_on_sample(ix, cents, cfg, args, pool_np, local_sizes, outs, time_it=False)
        ctx.set_option("time_kernels", 1)
        ctx.set_option("reset_timers", 1)
        for i in range(args.steps):
            ix.search_device(pool[i % len(pool)], npb, k, *o)
        torch.cuda.synchronize()
        st = ctx.stats()
        ctx.set_option("time_kernels", 0)
        n = max(1, st["timed_calls"])
        rows.append({"rank": r, "local_rows": info["local_rows"], "ms_per_step": round(ms, 4),
                     "assign_ms": round(st["assign_ms"] / n, 4), "scan_ms": round(st["scan_ms"] / n, 4),
                     "finalize_ms": round(st["finalize_ms"] / n, 4),
                     "striped_lists": info["shard"]["striped_lists"],
                     "parity_sample": parity and {kk: parity[kk] for kk in ("queries", "from_timed_batch",
                                                                          "bit_exact", "mismatched_queries")}})
        log(f"shard {r}/{N}: {rows[-1]}")
        ix.close()
        del ix
        torch.cuda.empty_cache()
    worst = max(x["ms_per_step"] for x in rows)
    line = {"metric": METRIC + " -- per-shard local search of an N-GPU job on one GPU",
            "value": round(B / (worst / 1e3), 2), "unit": UNIT, "n_gpus": 1, "steps": args.steps,
            "warmup": args.warmup, "higher_is_better": True,
            "config": config_dict(cfg, args),
            "shards": rows, "n_shards": N,
            "spread": {"min_ms": min(x["ms_per_step"] for x in rows), "max_ms": worst,
                       "mean_ms": round(float(np.mean([x["ms_per_step"] for x in rows])), 4)},
            "compute_assignments_s": round(t_assign, 1),
            "note": "value = batch / slowest shard's local step (no exchange): an upper bound on the "
                    "N-GPU step rate; the full step adds the slice assign + two small all-gathers"}
    print(json.dumps(line), flush=True)


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
    ix, cents, sizes, local_sizes, owner, assign, _ = build_index(wl, ctx, 0, 1)
    k = max(cfg.k, c5.K_CACHE)
    Qpool = torch.cat([wl.queries(1000 + i) for i in range(8)]).cpu().numpy()
    budget = int(64 * sizes.mean())  # ~64 lists of rows per sub-stage
    levels = [int(x) for x in os.environ.get("HIVF_C5_LEVELS", "1,8,64,256,512").split(",")]
    ref_ix = None
    if oracle.ref_available() and not args.no_cpu:
        t0 = time.time()
        ref_ix, _ = restricted_ref_index(ix, cents.cpu().numpy(), np.arange(cfg.k_clusters), local_sizes)
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


# ---------------------------------------------------------------------------
# reference arm
# ---------------------------------------------------------------------------

def run_c5_sched(args):
    """BASELINE.json configs[4] through the reference's UNMODIFIED scheduler:
    compat/_build/{gpu,cpu}/hedra_c5 (sched::run, LiveTransport) on a C2-shaped
    index (1M x 768, IVF-1024, nprobe 32), a 400-request HyDE / multistep /
    IRG mix.  --impl hivf runs the GPU engine (libhivf behind the reference
    API), --impl reference the reference's own retrieval engine (16 host
    threads) under the same scheduler and workload.  The line reports the
    retrieval sub-stage latency p50/p99 (the "substage" trace events) and the
    request latency p50/p99 of the ExperimentReport."""
    import subprocess
    if int(os.environ.get("RANK", "0")) != 0:
        return
    flavour = "cpu" if args.impl == "reference" else "gpu"
    exe = os.path.join(os.path.dirname(os.path.abspath(__file__)), "paper_2507_09138_b200", "compat", "_build",
                       flavour, "hedra_c5")
    if not os.path.exists(exe):
        print(json.dumps({"impl": args.impl, "unavailable": f"{exe} not built (compat/build.py)"}))
        return
    n_req = 400 if flavour == "gpu" else 100
    cmd = [exe, "--n", "1000000", "--dim", "768", "--topics", "256", "--clusters", "1024", "--spread", "0.03",
           "--requests", str(n_req), "--rate", "40", "--nprobe", "32", "--kmeans-sample", "48000",
           "--clock", "live", "--mix", "hyde=0.3,multistep=0.4,irg=0.3"]
    if flavour == "cpu":
        cmd += ["--kmeans-iters", "4"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        print(json.dumps({"impl": args.impl, "unavailable": r.stderr[-300:]}))
        return
    d = json.loads(r.stdout.strip().splitlines()[-1])
    line = {"metric": "C5 retrieval sub-stage latency under sched::run (live clock), p50", "value":
            d["substage_ms"]["p50"], "unit": "ms", "higher_is_better": False, "n_gpus": 1,
            "config": {"workload": "heterogeneous RAG stream (HyDE / multistep / IRG) through the reference scheduler",
                       "index": d["corpus"] + f" IVF-{d['clusters']}", "nprobe": d["nprobe"], "requests": d["requests"]},
            "substage_ms": d["substage_ms"], "items_per_substage": d["items_per_substage"],
            "request_latency_ms": {"p50": d["latency_p50_ms"], "p99": d["latency_p99_ms"]},
            "per_vector_ns": d["per_vector_ns"], "engine": d["engine"], "completed": d["completed"]}
    if args.impl == "reference":
        line["impl"] = "reference"
    print(json.dumps(line), flush=True)


def run_reference(args):
    """The reference's own CPU implementation (oracle/_ref: the unmodified
    /root/reference/proj sources compiled), rank 0 only, on the same workload,
    config and query sample as our arm's parity / cpu_baseline: per step one
    sample chunk (make_cursor x S + RetrievalEngine::execute(live_math=true),
    S >= host threads so every core works).  The index is the one
    index_from_assignments builds from the same centroids and the exact
    assignment (bench_workload.exact_assign: torch, no libhivf in this arm)."""
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
    assign = wl.exact_assign(cents)
    cents_np = cents.cpu().numpy()
    log(f"reference: centroids + exact assignments in {time.time() - t0:.1f}s")
    empty = oracle.RefIndex.from_csr(cents_np, np.zeros(cfg.k_clusters + 1, np.uint64),
                                     np.zeros((0, cfg.dim), np.float32), np.zeros(0, np.uint64))
    chunks = sample_plan(cfg, args)
    nproc = os.cpu_count() or 1
    steps_of = {c: [i for i in range(args.steps) if i % len(chunks) == c] for c in range(len(chunks))}
    times, qs = [], []
    for c, (j, first, S) in enumerate(chunks):
        if not steps_of[c] and c > 0:
            continue
        Q = wl.queries(j)[first:first + S].cpu().numpy()
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
            asg.append(a[m].cpu().numpy())
        rows, ids, asg = np.concatenate(rows), np.concatenate(ids), np.concatenate(asg)
        o = np.argsort(asg, kind="stable")  # index_from_assignments: lists in corpus order
        off = np.zeros(cfg.k_clusters + 1, np.uint64)
        off[1:] = np.cumsum(np.bincount(asg, minlength=cfg.k_clusters))
        ri = oracle.RefIndex.from_csr(cents_np, off, rows[o], ids[o])
        del rows, ids, asg, o
        log(f"reference: chunk {c} (batch {j} rows {first}:{first + S}): {int(off[-1])} rows")
        if c == 0:
            for _ in range(args.warmup):
                ri.bench_execute(Q, cfg.nprobe, cfg.k, live=True)
        for _ in steps_of[c]:
            ms, *_ = ri.bench_execute(Q, cfg.nprobe, cfg.k, live=True)
            times.append(ms)
            qs.append(S)
        del ri
    tot = sum(times)
    value = sum(qs) / (tot / 1e3)
    S_max = max(S for _, _, S in chunks)
    line = {
        "impl": "reference", "metric": METRIC, "value": round(value, 3), "unit": UNIT,
        "n_gpus": int(os.environ.get("WORLD_SIZE", "1")), "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(tot / len(times), 3),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32+f64",
        "data": "synthetic gaussian mixture (bench_workload.py)",
        "config": config_dict(cfg, args),
        "parallelism": f"{min(S_max, nproc)} host threads (RetrievalEngine::execute, one item per query)",
        "cpu_baseline": {"value": round(value, 3), "unit": UNIT, "cores": min(S_max, nproc),
                         "threads_used": min(S_max, nproc), "nproc": nproc, "cpu_model": cpu_model(),
                         "kind": "reference",
                         "sample": f"per step one of {len(chunks)} query chunks "
                                   f"({', '.join(f'{j}:{f}-{f + S}' for j, f, S in chunks)} of the pool "
                                   f"batches; full plans) on a restricted index of the chunk's probed lists"},
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
    ap.add_argument("--cpu-sample", type=int, default=16,
                    help="queries per reference chunk at C3/C4 (>= host threads)")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-graph", action="store_true", help="time direct launches instead of a CUDA graph")
    ap.add_argument("--hbm-budget-gb", type=float, default=0.0,
                    help="tiered residency: HBM bytes for list storage (rest in pinned host memory)")
    ap.add_argument("--shard", default="",
                    help="R/N or all/N: on one GPU, time rank R's (every rank's) list shard of an N-GPU job")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.cpu_sample < (os.cpu_count() or 1):
        log(f"note: --cpu-sample {args.cpu_sample} < {os.cpu_count()} host threads")
    if args.config == "c5":
        run_c5(args)
    elif args.config == "c5sched":
        run_c5_sched(args)
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
