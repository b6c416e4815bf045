"""Synthetic IVF workloads for bench.py (bench infrastructure, not product).

Distribution follows the reference generator's design
(/root/reference/proj/src/workload.cpp:23-35,135-164): topic centers on the
unit sphere, point i belongs to topic i mod T, per-dim N(0, spread^2) noise,
doc_id = i; queries = topic center + the same noise, topics uniform
(workload.cpp:241-309 samples topics; Zipf for skewed streams).  Generated on
the GPU with torch's counter-based Philox generator, one fixed seed per
262144-row chunk, so any chunk can be regenerated bit-identically (the index
build regenerates chunks instead of holding the 64 GB corpus twice).

Centroids: k-means (Lloyd) on a sample, deterministic (fp64 segment sums) --
part of the synthetic input, like the corpus (both arms use the same ones).
Assignments: ivf::compute_assignments (vector_index.cpp:202-208; nearest
centroid by the reference's double distance, ties -> lowest id) over every
row.  Our arm computes them with the library (hivf_compute_assignments,
`library_assign`); the reference arm, which must not load our library, with
`exact_assign`, a torch restatement of the same arithmetic (fp32 GEMM filter
with a rigorous error bound, exact sequential double distances for the rows
the bound leaves ambiguous).  Both give the reference's assignment, so both
arms search the index index_from_assignments builds;
tests/test_gpu_build.py checks the two against each other and the oracle.
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np
import torch

CHUNK = 1 << 18


@dataclass
class Config:
    name: str
    n: int
    dim: int
    k_clusters: int
    nprobe: int
    k: int
    batch: int
    spread: float
    zipf: float = 0.0

    def describe(self) -> str:
        return (f"{self.n // 1_000_000 if self.n >= 1_000_000 else self.n}"
                f"{'M' if self.n >= 1_000_000 else ''}x{self.dim} IVF-{self.k_clusters} "
                f"nprobe={self.nprobe} k={self.k} batch={self.batch}")


CONFIGS = {
    # BASELINE.json configs[0..2] (configs[3]/[4] are multi-GPU / stream workloads)
    "c1": Config("c1", 100_000, 128, 256, 8, 10, 64, 0.25),
    "c2": Config("c2", 1_000_000, 768, 1024, 32, 10, 256, 0.03),
    "c3": Config("c3", 21_000_000, 768, 4096, 128, 10, 256, 0.03),
    # C3 index with a Zipf(1.0) topic-skewed query stream (residency experiments)
    "c3z": Config("c3z", 21_000_000, 768, 4096, 128, 10, 256, 0.03, zipf=1.0),
    # configs[3]: 100M x 768 (307 GB) IVF-16384 over 8 GPUs, Zipf(1.0) topic-skewed
    # queries (workload.cpp:168-183); nprobe unspecified in BASELINE -> 128
    "c4": Config("c4", 100_000_000, 768, 16384, 128, 10, 256, 0.03, zipf=1.0),
    # small configs for tests
    "tiny": Config("tiny", 60_000, 64, 64, 8, 10, 48, 0.3),
}


class Workload:
    def __init__(self, cfg: Config, device="cuda", corpus_seed=1, query_seed=2):
        self.cfg = cfg
        self.device = torch.device(device)
        self.corpus_seed = corpus_seed
        self.query_seed = query_seed
        self.topics = max(1, cfg.k_clusters // 4)
        g = torch.Generator(device=self.device).manual_seed(corpus_seed)
        c = torch.randn(self.topics, cfg.dim, generator=g, device=self.device, dtype=torch.float64)
        c = c / c.norm(dim=1, keepdim=True).clamp_min(1e-300)
        self.centers = c.float()

    # -- corpus -----------------------------------------------------------------
    def n_chunks(self) -> int:
        return (self.cfg.n + CHUNK - 1) // CHUNK

    def chunk(self, ci: int) -> torch.Tensor:
        """Rows [ci*CHUNK, min(n, (ci+1)*CHUNK)) as a [rows, dim] float32 tensor."""
        first = ci * CHUNK
        rows = min(CHUNK, self.cfg.n - first)
        g = torch.Generator(device=self.device).manual_seed(self.corpus_seed * 1_000_003 + ci + 17)
        z = torch.randn(rows, self.cfg.dim, generator=g, device=self.device, dtype=torch.float32)
        topic = torch.arange(first, first + rows, device=self.device) % self.topics
        return self.centers[topic] + z * self.cfg.spread

    # -- queries ----------------------------------------------------------------
    def queries(self, batch_index: int, b: int | None = None) -> torch.Tensor:
        b = b or self.cfg.batch
        g = torch.Generator(device=self.device).manual_seed(self.query_seed * 7919 + batch_index)
        if self.cfg.zipf > 0:
            w = 1.0 / torch.arange(1, self.topics + 1, device=self.device,
                                   dtype=torch.float64) ** self.cfg.zipf
            t = torch.multinomial(w, b, replacement=True, generator=g)
        else:
            t = torch.randint(0, self.topics, (b,), generator=g, device=self.device)
        z = torch.randn(b, self.cfg.dim, generator=g, device=self.device, dtype=torch.float32)
        return (self.centers[t] + z * self.cfg.spread).contiguous()

    # -- centroids ----------------------------------------------------------------
    @staticmethod
    def _assign(x: torch.Tensor, cents: torch.Tensor, cn2: torch.Tensor) -> torch.Tensor:
        return torch.argmin(cn2[None, :] - 2.0 * (x @ cents.T), dim=1)

    def train_centroids(self, iters: int = 6, sample_per_centroid: int = 48) -> torch.Tensor:
        K = self.cfg.k_clusters
        want = min(self.cfg.n, max(K, sample_per_centroid * K))
        parts, got, ci = [], 0, 0
        while got < want:
            c = self.chunk(ci)[: want - got]
            parts.append(c)
            got += c.shape[0]
            ci += 1
        x = torch.cat(parts)
        g = torch.Generator(device=self.device).manual_seed(self.corpus_seed + 99)
        cents = x[torch.randperm(x.shape[0], generator=g, device=self.device)[:K]].clone()
        prev = torch.backends.cuda.matmul.allow_tf32
        torch.backends.cuda.matmul.allow_tf32 = False
        try:
            for _ in range(iters):
                a = self._assign(x, cents, (cents * cents).sum(1))
                order = torch.sort(a, stable=True).indices
                counts = torch.bincount(a, minlength=K)
                cs = torch.zeros(x.shape[0] + 1, x.shape[1], device=self.device, dtype=torch.float64)
                cs[1:] = torch.cumsum(x[order].double(), dim=0)
                ends = torch.cumsum(counts, 0)
                starts = ends - counts
                sums = cs[ends] - cs[starts]
                nz = counts > 0
                cents[nz] = (sums[nz] / counts[nz, None].double()).float()
        finally:
            torch.backends.cuda.matmul.allow_tf32 = prev
        return cents.contiguous()

    def library_assign(self, ctx, cents: torch.Tensor) -> torch.Tensor:
        """compute_assignments of every row through libhivf (hivf_compute_assignments)."""
        out = torch.empty(self.cfg.n, dtype=torch.int32, device=self.device)
        cents = cents.contiguous()
        for ci in range(self.n_chunks()):
            x = self.chunk(ci).contiguous()
            ctx.compute_assignments(x, cents, out[ci * CHUNK: ci * CHUNK + x.shape[0]])
        return out.long()

    def exact_assign(self, cents: torch.Tensor, sub: int = 32768) -> torch.Tensor:
        """compute_assignments restated in torch (bench infrastructure for the
        reference arm): nearest_centroid (vector_index.cpp:18-29) by the
        reference's squared_l2 (embedding.hpp:27-34), ties -> lowest id."""
        K, D = cents.shape
        c64 = cents.double()
        cnorm = c64.norm(dim=1)
        cn2 = (cents * cents).sum(1)
        out = torch.empty(self.cfg.n, dtype=torch.int64, device=self.device)
        # |fp32 GEMM distance - exact| <= (D+4) 2^-24 (|x|+|c|)^2 for any
        # summation order (FMA or not); x4 headroom
        gam = 4.0 * (D + 4) * 2.0 ** -24
        prev = torch.backends.cuda.matmul.allow_tf32
        torch.backends.cuda.matmul.allow_tf32 = False
        try:
            for ci in range(self.n_chunks()):
                xc = self.chunk(ci)
                for s0 in range(0, xc.shape[0], sub):
                    x = xc[s0:s0 + sub]
                    d = (x * x).sum(1, keepdim=True) + cn2[None, :] - 2.0 * (x @ cents.T)
                    xn = x.double().norm(dim=1)
                    E = (gam * (xn + cnorm.max()) ** 2).float()[:, None] * 1.0001 + 1e-30
                    best = d.min(dim=1).values
                    cand = d <= (best[:, None] + 2 * E)
                    n_c = cand.sum(1)
                    res = d.argmin(dim=1)
                    amb = torch.nonzero(n_c > 1).squeeze(1)
                    if amb.numel():
                        r, c = torch.nonzero(cand[amb], as_tuple=True)
                        xa = x[amb[r]].double()
                        ca = c64[c]
                        acc = torch.zeros(r.shape[0], dtype=torch.float64, device=self.device)
                        for i in range(D):  # sequential, one rounding per op, no FMA
                            t = xa[:, i] - ca[:, i]
                            acc = acc + t * t
                        # min (distance, id): ids ascending within a row after nonzero()
                        key_best = torch.full((amb.shape[0],), float("inf"), dtype=torch.float64,
                                              device=self.device)
                        key_best.scatter_reduce_(0, r, acc, reduce="amin")
                        hit = acc == key_best[r]
                        pick = torch.full((amb.shape[0],), K, dtype=torch.int64, device=self.device)
                        pick.scatter_reduce_(0, r[hit], c[hit], reduce="amin")
                        res[amb] = pick
                    out[ci * CHUNK + s0: ci * CHUNK + s0 + x.shape[0]] = res
        finally:
            torch.backends.cuda.matmul.allow_tf32 = prev
        return out


def list_layout(assign: torch.Tensor, k_clusters: int):
    """index_from_assignments order: list offsets + each row's list-order position."""
    counts = torch.bincount(assign, minlength=k_clusters)
    off = torch.zeros(k_clusters + 1, dtype=torch.int64, device=assign.device)
    off[1:] = torch.cumsum(counts, 0)
    order = torch.sort(assign, stable=True).indices
    pos = torch.empty_like(order)
    pos[order] = torch.arange(assign.shape[0], device=assign.device)
    return off, pos, order


def algorithmic_bytes(plans: np.ndarray, sizes: np.ndarray, dim: int, k_clusters: int, elem: int = 4) -> int:
    """distinct probed lists streamed once (elem bytes per
    element: 4 for the fp32 lists, 2 when the scan reads the fp16 filter copy)
    + centroids + queries."""
    uniq = np.unique(plans)
    return int(sizes[uniq].sum()) * elem * dim + k_clusters * 4 * dim + plans.shape[0] * 4 * dim


def list_bytes(plans: np.ndarray, sizes: np.ndarray, dim: int, elem: int = 4) -> int:
    return int(sizes[np.unique(plans)].sum()) * elem * dim


def human(n: float) -> str:
    for u in ["", "K", "M", "G", "T"]:
        if abs(n) < 1000:
            return f"{n:.3g}{u}"
        n /= 1000
    return f"{n:.3g}P"


__all__ = ["CHUNK", "CONFIGS", "Config", "Workload", "list_layout",
           "algorithmic_bytes", "list_bytes", "human", "math"]
