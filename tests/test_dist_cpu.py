"""Multi-process data parallelism on CPU (gloo, world size 2).

Covers the host-side N > 1 logic: batch sharding, the packed shared-gradient
layout and the single all-reduce. Each rank computes its shard's gradients
with the CPU checker (the device path is exercised by the -m gpu suite), packs
[sum dV, sum dw] exactly like mrf_pack_shared_grads_f32, all-reduces, and the
result must equal the single-process sum over the whole batch.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1910_10892_b200.dist import allreduce_shared, shard_range

B, H, W, L, CONN, K = 5, 6, 7, 4, 4, 2


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _problem(b):
    from oracle import oracle as O
    from paper_1910_10892_b200 import workloads as WL

    un, _, _, planes = WL.random_problem(H, W, L, CONN, seed=1000 + b, per_edge=True)
    _, V, _, _ = WL.random_problem(H, W, L, CONN, seed=7)  # shared pairwise table
    return O.Problem(H, W, L, CONN, un, V, 1.0, planes, 0.5, None)


def _image_grads(b):
    from oracle import oracle as O

    pr = _problem(b)
    f = O.forward("trwp", pr, K)
    gc = np.random.default_rng(b).normal(size=H * W * L).astype(np.float32)
    g = O.backward("trwp", pr, K, f.p, f.q, gc)
    return g.pairwise.astype(np.float64), float(g.wplanes.astype(np.float64).sum())


def _pack(images):
    dv = np.zeros(L * L)
    dw = 0.0
    for b in images:
        v, w = _image_grads(b)
        dv += v
        dw += w
    return torch.tensor(np.concatenate([dv, [dw]]), dtype=torch.float64)


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    start, stop = shard_range(B, rank, world)
    buf = _pack(range(start, stop))
    allreduce_shared(buf)
    out[rank] = buf.numpy().copy()
    dist.destroy_process_group()


def test_shard_range_partitions_batch():
    for batch in (1, 5, 8, 32, 33):
        for world in (1, 2, 4, 8):
            cover = []
            for rank in range(world):
                a, b = shard_range(batch, rank, world)
                cover.extend(range(a, b))
                assert b - a in (batch // world, batch // world + 1)
            assert cover == list(range(batch))
    with pytest.raises(ValueError):
        shard_range(4, 2, 2)


def test_gloo_world2_allreduce_matches_single_process():
    port = _free_port()
    manager = mp.Manager()
    out = manager.dict()
    mp.spawn(_worker, args=(2, port, out), nprocs=2, join=True)
    want = _pack(range(B)).numpy()
    for rank in range(2):
        got = out[rank]
        assert np.allclose(got, want, rtol=1e-12, atol=1e-12)


def test_seg_batch_shards_are_slices_of_the_batch():
    """A rank's C4 shard (workloads.seg_batch(first=...)) holds exactly the
    images the single-process batch holds at those positions, with the same
    shared pairwise table (bench.py --config C4 under torchrun)."""
    from paper_1910_10892_b200 import workloads as WL

    full = WL.seg_batch(12, 10, 5, 7)
    for world in (2, 3, 4):
        for rank in range(world):
            a, b = shard_range(7, rank, world)
            part = WL.seg_batch(12, 10, 5, b - a, first=a)
            assert np.array_equal(part.unary, full.unary[a:b])
            assert np.array_equal(part.w_planes, full.w_planes[a:b])
            assert np.array_equal(part.V, full.V)
