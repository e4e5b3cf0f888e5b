"""Multi-process (world_size 2, gloo on CPU) coverage of the N>1 path.

The real path runs one process per B200 with NCCL; here the same partitioning
and record gather run over gloo, with the per-rank "device run" replaced by the
CPU oracle — a test-only mock (the product has no CPU fallback).  Checks:
the global checksum is bitwise identical for W = 1 and W = 2 (SURVEY.md §8(e),
O11 batch independence), and every rank's slice is the right one.
"""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

import jm_synth
from paper_1904_08555_b200 import shard

N, DT, R, GLOBAL_BATCH, SEED = 5, "f64", 3, 37, 0x0019040855


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _rank_checksum(rank, world, strong=True, per_rank=11):
    import oracle
    first, cnt = (shard.strong_slice(rank, world, GLOBAL_BATCH) if strong
                  else shard.weak_slice(rank, per_rank))
    x = jm_synth.generate(N, DT, "bench", SEED, first, cnt)
    y = oracle.run(x, R, threads=1)          # mock of jit_mat_run on this rank's GPU
    return first, cnt, jm_synth.checksum(y, N, first)


def _worker(rank, world, port, q, strong):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    first, cnt, ck = _rank_checksum(rank, world, strong)
    recs, cks = shard.gather_record(dist, [float(first), float(cnt), 1.5 * rank], [ck], "cpu")
    if rank == 0:
        q.put((recs, [c[0] for c in cks]))
    dist.barrier()
    dist.destroy_process_group()


def _blob_worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    blob = bytes(range(256)) * 37 + b"JMC2" if rank == 0 else None
    got = shard.broadcast_blob(dist, blob, 0, "cpu")
    q.put((rank, got))
    dist.barrier()
    dist.destroy_process_group()


def test_world2_gloo_broadcasts_cache_blob():
    """f2: rank 0's compiled-kernel blob reaches every rank byte for byte."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_blob_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    got = dict(q.get(timeout=120) for _ in range(2))
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    want = bytes(range(256)) * 37 + b"JMC2"
    assert got[0] == want and got[1] == want


def _run_world(world, strong=True):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, world, port, q, strong)) for r in range(world)]
    for p in ps:
        p.start()
    out = q.get(timeout=120)
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    return out


def test_strong_slices_partition_the_batch():
    for world in (1, 2, 3, 4, 8):
        spans = [shard.strong_slice(r, world, GLOBAL_BATCH) for r in range(world)]
        assert spans[0][0] == 0
        assert sum(c for _, c in spans) == GLOBAL_BATCH
        for (a, ca), (b, _) in zip(spans, spans[1:]):
            assert a + ca == b
    with pytest.raises(ValueError):
        shard.strong_slice(2, 2, 10)


def test_checksum_combination_wraps():
    assert shard.combine_checksums([(1 << 64) - 1, 2]) == 1


def test_world2_gloo_matches_world1():
    recs, cks = _run_world(2)
    assert [r[:2] for r in recs] == [[0.0, 18.0], [18.0, 19.0]]
    assert recs[1][2] == 1.5
    whole = jm_synth.checksum(
        __import__("oracle").run(jm_synth.generate(N, DT, "bench", SEED, 0, GLOBAL_BATCH), R),
        N, 0)
    assert shard.combine_checksums(cks) == whole
    _, cks1 = _run_world(1)
    assert shard.combine_checksums(cks1) == whole


def test_world2_gloo_weak_scaling_slices():
    recs, cks = _run_world(2, strong=False)
    assert [r[:2] for r in recs] == [[0.0, 11.0], [11.0, 11.0]]
    x = jm_synth.generate(N, DT, "bench", SEED, 0, 22)
    y = __import__("oracle").run(x, R)
    assert shard.combine_checksums(cks) == jm_synth.checksum(y, N, 0)
    # per-rank pieces are themselves independent of how the batch was sliced
    assert np.array_equal(y[11:], __import__("oracle").run(jm_synth.generate(N, DT, "bench", SEED, 11, 11), R))
