"""Multi-rank host logic on CPU: the row-band plan, the gloo halo exchange and assembly
(world_size 2 and 3, real torch.distributed processes), and batch sharding by global image
index.  Compute stages use the oracle test double (tests/band_oracle_backend.py)."""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import synth
from paper_1505_00996_b200 import bands


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("H,W,r,s,world", [(64, 48, 4, 2, 2), (100, 40, 8, 4, 3), (4096, 64, 32, 4, 8),
                                           (16384, 16, 32, 4, 8), (101, 40, 8, 4, 3),
                                           (253, 364, 4, 4, 6)])
def test_band_plan_tiles_the_image(H, W, r, s, world):
    plans = [bands.plan_band(H, W, r, s, world, k) for k in range(world)]
    assert plans[0].Y0 == 0 and plans[-1].Y1 == H
    for a, b in zip(plans, plans[1:]):
        assert a.Y1 == b.Y0 and a.y1 == b.y0 and b.Y0 % s == 0
    for pl in plans:
        # one extra row when h s != H: the map scale h / H > 1 / s reaches low-res row y1 + 1
        x = int(pl.h * s != H)
        assert pl.halo == 2 * pl.R + 1 + x == 2 * oracle.radius_lowres(r, s) + 1 + x
        assert pl.e0 == max(0, pl.y0 - pl.halo) and pl.e1 == min(pl.h, pl.y1 + pl.halo)


def test_band_plan_rejects_thin_bands():
    with pytest.raises(ValueError):
        bands.plan_band(64, 64, 32, 4, 8, 0)   # 2 low-res rows per band < halo 17


def _image(H, W, C, seed):
    g = torch.Generator().manual_seed(seed)
    return torch.rand((1, C, H, W), generator=g, dtype=torch.float32)


@pytest.mark.parametrize("C_I,sub,H", [(1, 0, 90), (3, 1, 90), (1, 0, 89), (3, 1, 88)])
def test_local_band_simulation_matches_whole_image(C_I, sub, H):
    """H = 89, 88: not multiples of s, so the last rows of a band upsample from the low-res row
    after the band (the halo grows by one row; found by the GPU band fuzz)."""
    from tests.band_oracle_backend import OracleBackend
    W, r, s, eps = 52, 6, 3, 0.01
    I = _image(H, W, C_I, 1)
    p = _image(H, W, 2, 2)
    ref = oracle.fast_guided_filter(I.numpy(), p.numpy(), r, eps, s, sub)
    for world in (2, 3):
        q = bands.filter_bands_local(I, p, r, eps, s, sub, world, backend=OracleBackend())
        assert float(np.abs(q.numpy() - ref).max()) < 1e-6


@pytest.mark.parametrize("sub", [0, 1])
def test_local_bands_when_H_is_not_a_multiple_of_s(sub):
    """H = 4 h - 3 at s = 4: the map scale h / H exceeds 1 / s by the most, and the last rows of
    the bands ending below ~5/6 of the image upsample from the low-res row after the band --
    the halo carries one more row (found by the GPU band fuzz, seed 153)."""
    from tests.band_oracle_backend import OracleBackend
    H, W, r, s, eps, world = 253, 60, 4, 4, 1e-3, 8
    I = _image(H, W, 1, 3)
    p = _image(H, W, 2, 4)
    ref = oracle.fast_guided_filter(I.numpy(), p.numpy(), r, eps, s, sub)
    q = bands.filter_bands_local(I, p, r, eps, s, sub, world, backend=OracleBackend())
    assert float(np.abs(q.numpy() - ref).max()) < 1e-6


def _worker(rank, world, port, H, W, r, s, eps, sub, out_path):
    from tests.band_oracle_backend import OracleBackend
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    I = _image(H, W, 1, 7)
    p = _image(H, W, 1, 8)
    pl = bands.plan_band(H, W, r, s, world, rank)
    q = bands.filter_band(I[:, :, pl.Y0:pl.Y1].contiguous(), p[:, :, pl.Y0:pl.Y1].contiguous(), r,
                          eps, s, sub, H, rank, world, bands.DistExchange(rank, world),
                          backend=OracleBackend())
    parts = [None] * world
    dist.all_gather_object(parts, q.numpy())
    if rank == 0:
        np.save(out_path, np.concatenate(parts, axis=2))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world,H", [(2, 96), (3, 96), (3, 95)])
def test_gloo_band_exchange_matches_whole_image(tmp_path, world, H):
    W, r, s, eps, sub = 40, 6, 2, 0.02, 0
    out = str(tmp_path / "q.npy")
    mp.spawn(_worker, args=(world, _free_port(), H, W, r, s, eps, sub, out), nprocs=world,
             join=True)
    q = np.load(out)
    ref = oracle.fast_guided_filter(_image(H, W, 1, 7).numpy(), _image(H, W, 1, 8).numpy(), r, eps,
                                    s, sub)
    assert float(np.abs(q - ref).max()) < 1e-6


def _shard_worker(rank, world, port, out_path):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    B = 2  # images per rank (weak scaling: rank k owns global images [k B, (k+1) B))
    I, p = synth.make_batch(1, "cpu", batch=B, first=rank * B, H=48, W=64)
    q = oracle.fast_guided_filter(I.numpy(), p.numpy(), **synth.params(1))
    parts = [None] * world
    dist.all_gather_object(parts, q)
    if rank == 0:
        np.save(out_path, np.concatenate(parts, axis=0))
    dist.barrier()
    dist.destroy_process_group()


def test_gloo_batch_sharding_reproduces_single_process(tmp_path):
    out = str(tmp_path / "q.npy")
    mp.spawn(_shard_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    I, p = synth.make_batch(1, "cpu", batch=4, first=0, H=48, W=64)
    ref = oracle.fast_guided_filter(I.numpy(), p.numpy(), **synth.params(1))
    np.testing.assert_array_equal(np.load(out), ref)
