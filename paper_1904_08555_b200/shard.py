"""Batch partitioning and the per-rank record gather.

The update has no exchange step: every matrix is independent (PAPER.md:468,
"a proxy for part of a larger computation, presumably running on many
threads").  So multi-GPU is pure data parallelism over the batch:

* each rank owns a CONTIGUOUS slice of the global batch and generates its
  inputs from the GLOBAL matrix index (jit_mat_fill's ``global_first``), so the
  global result is identical for every world size;
* after the timed region, one collective gathers a small record per rank
  (timing, batch, checksum).  With NCCL this moves a few bytes over NVLink;
  with gloo it runs on CPU (tests/test_shard_gloo.py).

Host plumbing only — no arithmetic of the method lives here.
"""
from __future__ import annotations

MASK64 = (1 << 64) - 1


def strong_slice(rank: int, world: int, global_batch: int) -> tuple[int, int]:
    """Rank's [first, first+count) of a fixed global batch: floor(rB/W) split."""
    if not (0 <= rank < world) or global_batch < 0:
        raise ValueError("bad rank/world/batch")
    lo = rank * global_batch // world
    hi = (rank + 1) * global_batch // world
    return lo, hi - lo


def weak_slice(rank: int, per_rank: int) -> tuple[int, int]:
    """Rank's slice when every rank processes ``per_rank`` matrices (weak scaling)."""
    if rank < 0 or per_rank < 0:
        raise ValueError("bad rank/batch")
    return rank * per_rank, per_rank


def combine_checksums(values) -> int:
    """The global checksum is the per-rank u64 sums added mod 2^64 (order free)."""
    s = 0
    for v in values:
        s = (s + (int(v) & MASK64)) & MASK64
    return s


def _to_i64(u: int) -> int:
    u &= MASK64
    return u - (1 << 64) if u >= (1 << 63) else u


def gather_record(dist, floats: list[float], u64s: list[int], device) -> tuple[list[list[float]], list[list[int]]]:
    """All-gather one record per rank: ``floats`` (f64) and ``u64s`` (carried as i64).

    ``device`` is the tensor device the backend needs (cuda:k for NCCL, cpu for gloo).
    Returns per-rank lists ordered by rank.
    """
    import torch

    world = dist.get_world_size()
    f = torch.tensor(floats, dtype=torch.float64, device=device)
    fs = [torch.empty_like(f) for _ in range(world)]
    dist.all_gather(fs, f)
    if not u64s:
        return [t.cpu().tolist() for t in fs], [[] for _ in range(world)]
    u = torch.tensor([_to_i64(x) for x in u64s], dtype=torch.int64, device=device)
    us = [torch.empty_like(u) for _ in range(world)]
    dist.all_gather(us, u)
    return ([t.cpu().tolist() for t in fs],
            [[x & MASK64 for x in t.cpu().tolist()] for t in us])


def broadcast_blob(dist, blob: bytes | None, src: int, device) -> bytes:
    """Broadcast a byte string (a jit_mat_cache_export blob) from rank ``src``.

    SURVEY.md §8(f) f2: one rank runs NVRTC, the others install its cubins
    with jit_mat_cache_import, so W ranks compile each key once instead of W
    times (the paper's "maximal reuse of compiler state").  Two
    collectives: the length, then the bytes (as uint8 on ``device``).
    """
    import torch

    rank = dist.get_rank()
    n = torch.tensor([len(blob) if rank == src else 0], dtype=torch.int64, device=device)
    dist.broadcast(n, src)
    buf = (torch.frombuffer(bytearray(blob), dtype=torch.uint8).to(device) if rank == src
           else torch.empty(int(n.item()), dtype=torch.uint8, device=device))
    dist.broadcast(buf, src)
    return bytes(buf.cpu().numpy().tobytes())
