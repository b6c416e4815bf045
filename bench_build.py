"""Index-build timing (bench infrastructure): the library's index build on the
BASELINE workloads, written to gpurun_out/build_bench.json (committed copy
under profiles/).

  c1, c2  hivf_train_kmeans (the reference's train_kmeans, bit-identical:
          k-means++ seeding + Lloyd) and hivf_compute_assignments over every
          row; c1 also times the reference's own train_kmeans (oracle/_ref) on
          the host and checks the centroids bit for bit.
  c3      the whole 21M x 768 corpus in HBM (64.5 GB): the parallel training
          mode hivf_train_kmeans_sampled_seeds (K distinct rows drawn with the
          reference's Rng as seeds, then the reference's exact Lloyd
          iterations over all 21M rows) and compute_assignments of every row.
  c4      100M x 768 does not fit one GPU: sampled-seed training on a
          786K-row sample (48 rows per centroid), then compute_assignments of
          all 100M rows streamed through HBM in chunks.

    python bench_build.py [c1 c2 c3 c4]
"""
import json
import os
import sys
import time

sys.path.insert(0, os.getcwd())
import numpy as np
import torch

import oracle
from bench_workload import CHUNK, CONFIGS, Workload
from paper_2507_09138_b200 import Context


def sync_time():
    torch.cuda.synchronize()
    return time.perf_counter()


def full_corpus(wl, cfg):
    X = torch.empty(cfg.n, cfg.dim, device="cuda")
    for ci in range(wl.n_chunks()):
        x = wl.chunk(ci)
        X[ci * CHUNK: ci * CHUNK + x.shape[0]] = x
    return X


def small(name, iters, do_ref):
    cfg = CONFIGS[name]
    wl = Workload(cfg, device="cuda:0")
    X = full_corpus(wl, cfg)
    ctx = Context(0, torch.cuda.current_stream())
    cents = torch.empty(cfg.k_clusters, cfg.dim, device="cuda")
    ctx.train_kmeans(X[:1000].contiguous(), 8, 1, 1, cents[:8])  # warm
    t0 = sync_time()
    ctx.train_kmeans(X, cfg.k_clusters, iters, 1, cents)
    t1 = sync_time()
    asg = torch.empty(cfg.n, dtype=torch.int32, device="cuda")
    ctx.compute_assignments(X, cents, asg)
    t2 = sync_time()
    r = {"n": cfg.n, "dim": cfg.dim, "K": cfg.k_clusters, "iters": iters, "mode": "k-means++ (reference)",
         "gpu_train_kmeans_s": round(t1 - t0, 3), "gpu_compute_assignments_s": round(t2 - t1, 4)}
    if do_ref:
        Xh = X.cpu().numpy()
        t3 = time.perf_counter()
        ref = oracle.ref_train_kmeans(Xh, cfg.k_clusters, iters, 1)
        r["ref_train_kmeans_s"] = round(time.perf_counter() - t3, 2)
        r["bit_exact"] = bool(np.array_equal(ref.view(np.uint32), cents.cpu().numpy().view(np.uint32)))
    return r


def c3(iters=4):
    cfg = CONFIGS["c3"]
    wl = Workload(cfg, device="cuda:0")
    t0 = sync_time()
    X = full_corpus(wl, cfg)
    t1 = sync_time()
    ctx = Context(0, torch.cuda.current_stream())
    cents = torch.empty(cfg.k_clusters, cfg.dim, device="cuda")
    ctx.train_kmeans_sampled_seeds(X, cfg.k_clusters, iters, 1, cents)
    t2 = sync_time()
    asg = torch.empty(cfg.n, dtype=torch.int32, device="cuda")
    ctx.compute_assignments(X, cents, asg)
    t3 = sync_time()
    sizes = torch.bincount(asg.long(), minlength=cfg.k_clusters)
    return {"n": cfg.n, "dim": cfg.dim, "K": cfg.k_clusters, "iters": iters,
            "mode": "sampled seeds (reference Rng) + exact Lloyd over every row",
            "generate_s": round(t1 - t0, 2), "gpu_train_kmeans_s": round(t2 - t1, 2),
            "gpu_compute_assignments_s": round(t3 - t2, 2),
            "list_sizes": {"min": int(sizes.min()), "max": int(sizes.max()), "empty": int((sizes == 0).sum())}}


def c4(iters=6, per_centroid=48):
    cfg = CONFIGS["c4"]
    wl = Workload(cfg, device="cuda:0")
    want = per_centroid * cfg.k_clusters
    parts, got, ci = [], 0, 0
    while got < want:
        x = wl.chunk(ci)[: want - got]
        parts.append(x)
        got += x.shape[0]
        ci += 1
    S = torch.cat(parts).contiguous()
    ctx = Context(0, torch.cuda.current_stream())
    cents = torch.empty(cfg.k_clusters, cfg.dim, device="cuda")
    t0 = sync_time()
    ctx.train_kmeans_sampled_seeds(S, cfg.k_clusters, iters, 1, cents)
    t1 = sync_time()
    del S
    asg = torch.empty(cfg.n, dtype=torch.int32, device="cuda")
    for ci in range(wl.n_chunks()):
        x = wl.chunk(ci).contiguous()
        ctx.compute_assignments(x, cents, asg[ci * CHUNK: ci * CHUNK + x.shape[0]])
    t2 = sync_time()
    sizes = torch.bincount(asg.long(), minlength=cfg.k_clusters)
    return {"n": cfg.n, "dim": cfg.dim, "K": cfg.k_clusters, "iters": iters, "sample_rows": want,
            "mode": "sampled seeds (reference Rng) + exact Lloyd on the sample",
            "gpu_train_kmeans_s": round(t1 - t0, 2),
            "gpu_compute_assignments_s": round(t2 - t1, 2),
            "compute_assignments_note": "includes generating the 100M rows chunk by chunk on device",
            "list_sizes": {"min": int(sizes.min()), "max": int(sizes.max()), "empty": int((sizes == 0).sum())}}


if __name__ == "__main__":
    which = sys.argv[1:] or ["c1", "c2"]
    out = {}
    os.makedirs("gpurun_out", exist_ok=True)
    for name in which:
        if name == "c1":
            out[name] = small("c1", 10, True)
        elif name == "c2":
            out[name] = small("c2", 3, False)
        elif name == "c3":
            out[name] = c3()
        elif name == "c4":
            out[name] = c4()
        print(json.dumps({name: out[name]}), flush=True)
        torch.cuda.empty_cache()
        json.dump(out, open("gpurun_out/build_bench.json", "w"), indent=1)
