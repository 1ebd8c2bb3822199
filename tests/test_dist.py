"""Multi-GPU sharding logic on CPU (gloo, world_size 2): unit assignment
covers every (view, tile) exactly once with equal padded lists, and the
gather -> unpack plumbing of dist.render_sharded rebuilds every pixel.
The render/unpack callables here are CPU stand-ins that encode each pixel's
own coordinates; the CUDA kernels behind them are covered by -m gpu tests."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2204_11762_b200 import dist as D


@pytest.mark.parametrize("mode", ["auto", "views", "rows", "diagonal"])
def test_assign_units_cover_and_balance(mode):
    for V, W, H, G in [(1, 64, 64, 1), (3, 100, 75, 2), (16, 480, 270, 8), (2, 17, 33, 4), (1, 2048, 2048, 8)]:
        lists = D.assign_units(V, W, H, G, mode)
        assert len(lists) == G and len({len(x) for x in lists}) == 1
        allu = np.concatenate(lists)
        real = allu[allu[:, 0] >= 0]
        tx, ty = D.tile_grid(W, H)
        assert len(real) == V * tx * ty
        keys = {tuple(r) for r in real}
        assert len(keys) == len(real)                      # no duplicates
        counts = [int((x[:, 0] >= 0).sum()) for x in lists]
        m = D.pick_mode(V, G) if mode == "auto" else mode
        if m == "diagonal":
            assert max(counts) - min(counts) <= 1          # balanced to one tile
        elif m == "views":
            per_view = tx * ty
            assert max(counts) - min(counts) <= per_view   # balanced to one view
            for r, x in enumerate(lists):                  # rank r owns views r, r+G, ...
                assert set(x[x[:, 0] >= 0][:, 0].tolist()) <= set(range(r, V, G))
        else:
            band = V * tx * D.SUPERTILE                     # one supertile row of every view
            assert max(counts) - min(counts) <= band


def test_rank_lists_keep_the_single_gpu_order():
    """Each rank's list is a subsequence of the 1-GPU supertile order, so a
    rank's kernel visits neighbouring tiles back to back (the locality the
    render kernel depends on)."""
    V, W, H = 3, 200, 120
    full = D.supertile_order(range(V), W, H)
    pos = {tuple(u): i for i, u in enumerate(full)}
    assert len(pos) == len(full) == V * np.prod(D.tile_grid(W, H))
    for mode in ("views", "rows"):
        for x in D.assign_units(V, W, H, 2, mode, pad=False):
            idx = [pos[tuple(u)] for u in x]
            assert idx == sorted(idx)
    # the supertile order itself: 2x2 tiles, row-major inside, supertiles row-major
    o = D.supertile_order([0], 64, 48).tolist()
    assert o[:8] == [[0, 0, 0], [0, 1, 0], [0, 0, 1], [0, 1, 1], [0, 2, 0], [0, 3, 0], [0, 2, 1], [0, 3, 1]]


def _fake_render(tiles):
    t = tiles.numpy()
    out = np.zeros((len(t), 16, 16, 4), np.float32)
    for i, (v, tx, ty) in enumerate(t):
        if v < 0:
            continue
        ys, xs = np.meshgrid(np.arange(16), np.arange(16), indexing="ij")
        out[i, :, :, 0] = v
        out[i, :, :, 1] = tx * 16 + xs
        out[i, :, :, 2] = ty * 16 + ys
        out[i, :, :, 3] = 1.0
    return torch.from_numpy(out)


def _fake_unpack(V, W, H):
    def unpack(packed, tiles):
        img = np.zeros((V, H, W, 4), np.float32)
        p = packed.numpy()
        for i, (v, tx, ty) in enumerate(tiles.numpy()):
            if v < 0:
                continue
            x0, y0 = tx * 16, ty * 16
            h, w = min(16, H - y0), min(16, W - x0)
            img[v, y0:y0 + h, x0:x0 + w] = p[i, :h, :w]
        return torch.from_numpy(img)
    return unpack


def _worker(rank, world, port, V, W, H, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    img, n = D.render_sharded(_fake_render, _fake_unpack(V, W, H), V, W, H, rank, world)
    if rank == 0:
        q.put(img.numpy())
    dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("V,W,H", [(2, 100, 75), (1, 48, 32)])
def test_render_sharded_gloo_world2(V, W, H):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, V, W, H, q)) for r in range(2)]
    for p in procs:
        p.start()
    img = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    ys, xs = np.meshgrid(np.arange(H), np.arange(W), indexing="ij")
    for v in range(V):
        np.testing.assert_array_equal(img[v, :, :, 0], v)
        np.testing.assert_array_equal(img[v, :, :, 1], xs)
        np.testing.assert_array_equal(img[v, :, :, 2], ys)
        np.testing.assert_array_equal(img[v, :, :, 3], 1.0)


def _view_worker(rank, world, port, V, H, W, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    img0 = torch.full((V, H, W, 4), -1.0) if rank == 0 else None
    bufs = [torch.empty((H, W, 4)) for _ in range(2)] if rank else None
    rendered = []

    def render_view(v, out):
        assert v % world == rank                       # only this rank's views
        out.copy_(torch.arange(H * W * 4, dtype=torch.float32).view(H, W, 4) + 1000.0 * v)
        rendered.append(v)

    for _ in range(2):                                  # two steps reuse the buffers
        for wk in D.gather_views_nccl(render_view, img0, V, rank, world, bufs=bufs):
            wk.wait()
    assert rendered == D.rank_views(V, world, rank) * 2
    if rank == 0:
        q.put(img0.numpy())
    dist.destroy_process_group()


@pytest.mark.parametrize("V", [5, 2])
def test_gather_views_world2(V):
    """The per-view gather schedule (dist.gather_views_nccl; NCCL on GPUs,
    gloo here): every view arrives in rank 0's image slot; the sender's two
    buffers are reused only after their sends completed."""
    H, W = 6, 5
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_view_worker, args=(r, 2, port, V, H, W, q)) for r in range(2)]
    for p in procs:
        p.start()
    img = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    base = np.arange(H * W * 4, dtype=np.float32).reshape(H, W, 4)
    for v in range(V):
        np.testing.assert_array_equal(img[v], base + 1000.0 * v)
