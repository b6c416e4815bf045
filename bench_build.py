"""Index-build timing (bench infrastructure): GPU hivf_train_kmeans / hivf_compute_assignments
on the C1/C2 workloads vs the reference train_kmeans (oracle/_ref) on the host; writes
gpurun_out/build_bench.json (committed copy: profiles/r1_index_build.json)."""
import sys, os, time, json
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import oracle
from bench_workload import CONFIGS, Workload
from paper_2507_09138_b200 import Context
out = {}
for name, iters, do_ref in [("c1", 10, True), ("c2", 3, False)]:
    cfg = CONFIGS[name]
    wl = Workload(cfg, device="cuda:0")
    X = torch.cat([wl.chunk(i) for i in range(wl.n_chunks())])[: cfg.n].contiguous()
    ctx = Context(0, torch.cuda.current_stream())
    cents = torch.empty(cfg.k_clusters, cfg.dim, device="cuda")
    ctx.train_kmeans(X[:1000].contiguous(), 8, 1, 1, cents[:8])  # warm
    torch.cuda.synchronize(); t0 = time.perf_counter()
    ctx.train_kmeans(X, cfg.k_clusters, iters, 1, cents)
    torch.cuda.synchronize(); t1 = time.perf_counter()
    asg = torch.empty(cfg.n, dtype=torch.int32, device="cuda")
    ctx.compute_assignments(X, cents, asg); torch.cuda.synchronize(); t2 = time.perf_counter()
    r = {"n": cfg.n, "dim": cfg.dim, "K": cfg.k_clusters, "iters": iters,
         "gpu_train_kmeans_s": round(t1 - t0, 3), "gpu_compute_assignments_s": round(t2 - t1, 4)}
    if do_ref:
        Xh = X.cpu().numpy()
        t3 = time.perf_counter(); ref = oracle.ref_train_kmeans(Xh, cfg.k_clusters, iters, 1); t4 = time.perf_counter()
        r["ref_train_kmeans_s"] = round(t4 - t3, 2)
        r["bit_exact"] = bool(np.array_equal(ref.view(np.uint32), cents.cpu().numpy().view(np.uint32)))
    out[name] = r
    print(json.dumps(r), flush=True)
json.dump(out, open("gpurun_out/build_bench.json", "w"))
