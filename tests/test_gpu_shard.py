"""Multi-GPU list sharding through the library (hivf_group_*), on one GPU.

The driver's boxes have one B200, so the N-rank path runs with N contexts on
device 0 -- the exact code of an N-GPU job with the exchange between members
on the same device:
  * in-process group (hivf_group_create): one thread, N contexts, the gather
    kernel over peer pointers;
  * host-callback group (hivf_group_create_hostcb): N processes on one GPU,
    all-gathers through torch.distributed (gloo) -- the per-rank code path
    of the NCCL transport with a different exchange primitive;
  * NCCL group with one rank (NCCL refuses two ranks on one device): dlopen,
    communicator init and ncclAllGather on the context stream.
Every result is compared bit-for-bit with the oracle's unsharded search
(make_cursor + search_step, vector_index.cpp:280-328), which equals
merge_topk (:71-91) over the shards."""
import os
import socket

import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu


def _data(seed=5, n=40000, dim=96, K=64, B=37):
    rng = np.random.default_rng(seed)
    centers = rng.standard_normal((16, dim)).astype(np.float32)
    X = (centers[np.arange(n) % 16] + 0.3 * rng.standard_normal((n, dim))).astype(np.float32)
    cents = X[rng.choice(n, K, replace=False)].copy()
    assign = oracle.compute_assignments(X, cents)
    ids = rng.permutation(n).astype(np.uint64) * 3 + 7
    full = oracle.CsrIndex.from_assignments(X, ids, cents, assign)
    Q = (centers[rng.integers(0, 16, B)] + 0.3 * rng.standard_normal((B, dim))).astype(np.float32)
    return full, Q


def _eq(got, want):
    gi, gd, gc = got
    oi, od, oc = want
    assert np.array_equal(gc, oc)
    assert np.array_equal(gi, oi)
    assert np.array_equal(gd.view(np.uint64), od.view(np.uint64))


def _shards(full, world, n_striped, weights=None):
    from paper_2507_09138_b200 import Context, shard_plan, upload_shard
    sizes = (full.off[1:] - full.off[:-1]).astype(np.uint64)
    owner = shard_plan(sizes, world, weights=weights, n_striped=n_striped)
    ctxs = [Context(0) for _ in range(world)]
    shards = [upload_shard(ctxs[r], full.centroids, full.off, full.vectors, full.ids, owner, world, r)
              for r in range(world)]
    return ctxs, shards, owner


@pytest.mark.parametrize("world,n_striped", [(2, 0), (2, 6), (3, -1), (4, 64)])
@pytest.mark.parametrize("nprobe,k", [(8, 10), (64, 20), (1, 5)])
def test_in_process_group_equals_oracle(world, n_striped, nprobe, k):
    from paper_2507_09138_b200 import ShardGroup
    full, Q = _data()
    ctxs, shards, owner = _shards(full, world, n_striped)
    g = ShardGroup.in_process(shards)
    want = full.search(Q, nprobe, k)
    _eq(g.search(Q, nprobe, k), want)
    _eq(g.search(Q, nprobe, k), want)  # second call: buffer reuse / event ordering
    # device variant, asynchronous on member 0's stream
    import torch
    torch.cuda.set_device(0)
    dq = torch.from_numpy(Q).cuda()
    ids = torch.zeros(Q.shape[0], k, dtype=torch.int64, device="cuda")
    d = torch.zeros(Q.shape[0], k, dtype=torch.float64, device="cuda")
    c = torch.zeros(Q.shape[0], dtype=torch.int32, device="cuda")
    for _ in range(3):
        g.search_device(dq, nprobe, k, ids, d, c)
    ctxs[0].synchronize()
    _eq((ids.cpu().numpy().view(np.uint64), d.cpu().numpy(), c.cpu().numpy().view(np.uint32)), want)
    g.close()


def test_in_process_group_edge_cases():
    """fewer queries than ranks, nprobe = K, k above the rows probed, weights."""
    from paper_2507_09138_b200 import InvalidArgument, ShardGroup
    full, Q = _data(seed=9, n=3000, dim=24, K=40, B=5)
    w = np.linspace(1.0, 50.0, 40)
    ctxs, shards, owner = _shards(full, 3, -1, weights=w)
    g = ShardGroup.in_process(shards)
    for B in (1, 2, 5):
        for nprobe, k in ((40, 10), (1, 400), (3, 1)):
            _eq(g.search(Q[:B], nprobe, k), full.search(Q[:B], nprobe, k))
    with pytest.raises(InvalidArgument):
        g.search(Q, 41, 10)
    with pytest.raises(InvalidArgument):
        g.search(Q, 4, 0)
    g.close()


def test_nccl_group_single_rank():
    from paper_2507_09138_b200 import HivfError, ShardGroup, nccl_unique_id
    import torch  # loads torch's NCCL first, as under torchrun
    torch.cuda.init()
    full, Q = _data(seed=11)
    ctxs, shards, owner = _shards(full, 1, 0)
    try:
        uid = nccl_unique_id()
    except HivfError as e:  # pragma: no cover - image without NCCL
        pytest.skip(str(e))
    g = ShardGroup.nccl(shards[0], 1, 0, uid)
    _eq(g.search(Q, 16, 10), full.search(Q, 16, 10))
    g.close()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _hostcb_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch
    import torch.distributed as dist
    from paper_2507_09138_b200 import Context, ShardGroup, shard_plan, upload_shard
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        full, Q = _data(seed=13)
        sizes = (full.off[1:] - full.off[:-1]).astype(np.uint64)
        owner = shard_plan(sizes, world, n_striped=5)
        ctx = Context(0)
        shard = upload_shard(ctx, full.centroids, full.off, full.vectors, full.ids, owner, world, rank)

        def allgather(send: bytes) -> bytes:
            t = torch.frombuffer(bytearray(send), dtype=torch.uint8)
            out = [torch.empty_like(t) for _ in range(world)]
            dist.all_gather(out, t)
            return b"".join(bytes(o.numpy()) for o in out)

        g = ShardGroup.host_allgather(shard, world, rank, allgather)
        res = [g.search(Q, nprobe, k) for nprobe, k in ((8, 10), (64, 20))]
        if rank == 0:
            q.put(res)
        g.close()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_hostcb_group_processes_equal_oracle(world):
    import torch.multiprocessing as mp
    full, Q = _data(seed=13)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_hostcb_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    for (nprobe, k), got in zip(((8, 10), (64, 20)), res):
        _eq(got, full.search(Q, nprobe, k))
