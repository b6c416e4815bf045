"""Multi-GPU sharding logic on CPU (world_size 2, gloo): list sharding by LPT on
bytes (bench_workload.shard_lists), per-shard exact top-k, all_gather of
(ids, dists, counts), merge_topk (vector_index.cpp:71-91) == unsharded search.
The device-side merge kernel is covered in test_gpu_parity.py."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from bench_workload import shard_lists


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _data(seed=3, n=3000, dim=12, K=24):
    rng = np.random.default_rng(seed)
    X = rng.standard_normal((n, dim)).astype(np.float32)
    cents = X[rng.choice(n, K, replace=False)].copy()
    assign = oracle.compute_assignments(X, cents)
    ids = rng.permutation(n).astype(np.uint64)
    Q = rng.standard_normal((20, dim)).astype(np.float32)
    return X, ids, cents, assign, Q


def _shard_csr(X, ids, cents, assign, owner, rank):
    """This rank's index: all centroids, only its own lists (others empty)."""
    mine = owner[assign] == rank
    K = cents.shape[0]
    a = np.asarray(assign, np.int64)[mine]
    order = np.argsort(a, kind="stable")
    off = np.zeros(K + 1, np.uint64)
    off[1:] = np.cumsum(np.bincount(a, minlength=K))
    return oracle.CsrIndex(cents, off, X[mine][order], ids[mine][order])


def _worker(rank, world, port, nprobe, k, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        X, ids, cents, assign, Q = _data()
        sizes = np.bincount(assign, minlength=cents.shape[0])
        owner = shard_lists(sizes, world)
        csr = _shard_csr(X, ids, cents, assign, owner, rank)
        li, ld, lc = csr.search(Q, nprobe, k)
        gi = [torch.zeros(li.shape, dtype=torch.int64) for _ in range(world)]
        gd = [torch.zeros(ld.shape, dtype=torch.float64) for _ in range(world)]
        gc = [torch.zeros(lc.shape, dtype=torch.int64) for _ in range(world)]
        dist.all_gather(gi, torch.from_numpy(li.view(np.int64)))
        dist.all_gather(gd, torch.from_numpy(ld))
        dist.all_gather(gc, torch.from_numpy(lc.astype(np.int64)))
        if rank == 0:
            merged_i, merged_d = [], []
            for b in range(Q.shape[0]):
                acc = []
                for r in range(world):
                    c = int(gc[r][b])
                    part = [(int(gi[r][b, e].numpy().view(np.uint64)), float(gd[r][b, e]))
                            for e in range(c)]
                    acc = oracle.merge_topk(acc, part, k)
                merged_i.append([i for i, _ in acc])
                merged_d.append([d for _, d in acc])
            q.put((merged_i, merged_d))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("nprobe,k", [(4, 10), (24, 7), (1, 20)])
def test_sharded_search_equals_unsharded_gloo(nprobe, k):
    X, ids, cents, assign, Q = _data()
    full = oracle.CsrIndex.from_assignments(X, ids, cents, assign)
    oi, od, oc = full.search(Q, nprobe, k)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, nprobe, k, q)) for r in range(2)]
    for p in procs:
        p.start()
    mi, md = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for b in range(Q.shape[0]):
        assert mi[b] == [int(x) for x in oi[b][:oc[b]]]
        assert md[b] == [float(x) for x in od[b][:oc[b]]]


def test_shard_lists_balanced_and_total():
    sizes = np.array([100, 1, 50, 50, 30, 20, 0, 75])
    owner = shard_lists(sizes, 3)
    assert set(owner.tolist()) <= {0, 1, 2}
    loads = [sizes[owner == r].sum() for r in range(3)]
    assert sum(loads) == sizes.sum()
    assert max(loads) - min(loads) <= sizes.max()
