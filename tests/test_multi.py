"""Multi-GPU sharding logic on CPU (world_size 2, gloo): the library's shard
planner (hivf_shard_plan: frequency-weighted LPT + striped hot lists) and
per-rank CSR (hivf_shard_local_lists) -- host code of libhivf.so, callable
without a GPU -- then per-shard exact top-k, all_gather of (ids, dists,
counts), merge_topk (vector_index.cpp:71-91) == unsharded search.  The device
side (hivf_group_* over the three transports) is covered in
tests/test_gpu_shard.py."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from paper_2507_09138_b200 import SHARD_STRIPED, shard_local_lists, shard_plan


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


def _shard_csr(full, owner, world, rank):
    """This rank's index: all centroids, its local lists (others empty)."""
    loc, first = shard_local_lists(full.off, owner, world, rank)
    rows = np.concatenate([np.arange(first[c], first[c] + (loc[c + 1] - loc[c]), dtype=np.int64)
                           for c in range(len(owner))])
    return oracle.CsrIndex(full.centroids, loc, full.vectors[rows], full.ids[rows])


def _worker(rank, world, port, nprobe, k, n_striped, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        X, ids, cents, assign, Q = _data()
        full = oracle.CsrIndex.from_assignments(X, ids, cents, assign)
        sizes = np.bincount(assign, minlength=cents.shape[0])
        owner = shard_plan(sizes, world, n_striped=n_striped)
        csr = _shard_csr(full, owner, world, rank)
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


@pytest.mark.parametrize("nprobe,k,n_striped", [(4, 10, 0), (24, 7, 5), (1, 20, -1)])
def test_sharded_search_equals_unsharded_gloo(nprobe, k, n_striped):
    X, ids, cents, assign, Q = _data()
    full = oracle.CsrIndex.from_assignments(X, ids, cents, assign)
    oi, od, oc = full.search(Q, nprobe, k)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, nprobe, k, n_striped, q)) for r in range(2)]
    for p in procs:
        p.start()
    mi, md = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for b in range(Q.shape[0]):
        assert mi[b] == [int(x) for x in oi[b][:oc[b]]]
        assert md[b] == [float(x) for x in od[b][:oc[b]]]


def test_shard_plan_lpt_balance_and_striping():
    sizes = np.array([100, 1, 50, 50, 30, 20, 0, 75], np.uint64)
    owner = shard_plan(sizes, 3, n_striped=0)
    assert set(owner.tolist()) <= {0, 1, 2}
    loads = [int(sizes[owner == r].sum()) for r in range(3)]
    assert sum(loads) == int(sizes.sum())
    assert max(loads) - min(loads) <= int(sizes.max())
    # the heaviest list goes first, to rank 0 (LPT, ties to the lowest rank)
    assert owner[0] == 0
    # striping: the n heaviest by (load desc, id asc); weights scale the load
    owner = shard_plan(sizes, 3, n_striped=2)
    assert owner[0] == SHARD_STRIPED and owner[7] == SHARD_STRIPED
    w = np.ones(8)
    w[5] = 100.0
    owner = shard_plan(sizes, 3, weights=w, n_striped=1)
    assert owner[5] == SHARD_STRIPED and owner[0] != SHARD_STRIPED
    # auto: lists heavier than 1/16 of a rank's share are striped
    big = np.array([10_000] + [10] * 200, np.uint64)
    owner = shard_plan(big, 4, n_striped=-1)
    assert owner[0] == SHARD_STRIPED and (owner[1:] != SHARD_STRIPED).all()
    assert (shard_plan(sizes, 1) == 0).all()


@pytest.mark.parametrize("world", [1, 2, 3, 8])
def test_shard_local_lists_partition_rows(world):
    rng = np.random.default_rng(world)
    sizes = rng.integers(0, 40, 30).astype(np.uint64)
    off = np.zeros(31, np.uint64)
    off[1:] = np.cumsum(sizes)
    owner = shard_plan(sizes, world, n_striped=4 if world > 1 else 0)
    seen = np.zeros(int(off[-1]), np.int64)
    for r in range(world):
        loc, first = shard_local_lists(off, owner, world, r)
        for c in range(30):
            n = int(loc[c + 1] - loc[c])
            assert off[c] <= first[c] and first[c] + n <= off[c + 1]
            seen[int(first[c]):int(first[c]) + n] += 1
            if owner[c] not in (r, SHARD_STRIPED):
                assert n == 0
    assert (seen == 1).all()  # every row on exactly one rank
