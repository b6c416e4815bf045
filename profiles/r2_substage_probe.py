"""Latency of one node-split sub-stage (hivf_scan_items) on the C2 index as
the C5 scheduler issues them (4 items x 32 clusters, k = 20): wall time per
call and the library's phase split (time_kernels)."""
import os, sys, time, json
sys.path.insert(0, os.getcwd())
import numpy as np, torch
from bench_workload import CONFIGS, Workload
from paper_2507_09138_b200 import Context
import bench
cfg = CONFIGS["c2"]
torch.cuda.set_device(0)
wl = Workload(cfg, device="cuda:0")
ctx = Context(0, torch.cuda.current_stream())
ix, cents, sizes, local_sizes, owner, assign, info = bench.build_index(wl, ctx, 0, 1)
Q = wl.queries(0).cpu().numpy()
plans = ix.select_clusters(Q[:64], cfg.nprobe)
out = {}
for n_items, per in ((1, 32), (4, 8), (4, 32), (16, 32), (64, 32)):
    off = np.arange(n_items + 1, dtype=np.uint32) * per
    cl = np.concatenate([plans[i, :per] for i in range(n_items)]).astype(np.uint32)
    k = np.full(n_items, 20, np.uint32)
    ts = []
    for r in range(30):
        hid = np.zeros((n_items, 20), np.uint64); hd = np.zeros((n_items, 20)); hn = np.zeros(n_items, np.uint32)
        t0 = time.perf_counter()
        ix.scan_items(Q[:n_items], off, cl, k, hid, hd, hn)
        ts.append(time.perf_counter() - t0)
    ctx.set_option("time_kernels", 1); ctx.set_option("reset_timers", 1)
    for r in range(10):
        hid = np.zeros((n_items, 20), np.uint64); hd = np.zeros((n_items, 20)); hn = np.zeros(n_items, np.uint32)
        ix.scan_items(Q[:n_items], off, cl, k, hid, hd, hn)
    st = ctx.stats(); ctx.set_option("time_kernels", 0)
    ts = sorted(ts[5:])
    out[f"{n_items}x{per}"] = {"wall_ms_p50": round(1e3 * ts[len(ts) // 2], 4), "wall_ms_min": round(1e3 * ts[0], 4),
                               "scan_ms": round(st["scan_ms"] / max(1, st["timed_calls"]), 4),
                               "finalize_ms": round(st["finalize_ms"] / max(1, st["timed_calls"]), 4),
                               "kernels": st["kernels_launched"], "group": st["scan_group"]}
    print(f"{n_items}x{per}", out[f"{n_items}x{per}"], flush=True)
json.dump(out, open("gpurun_out/substage_probe.json", "w"), indent=1)
