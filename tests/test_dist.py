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


def test_assign_units_cover_and_balance():
    for V, W, H, G in [(1, 64, 64, 1), (3, 100, 75, 2), (64, 3840, 2160, 8), (2, 17, 33, 4)]:
        lists = D.assign_units(V, W, H, G)
        assert len(lists) == G and len({len(x) for x in lists}) == 1
        allu = np.concatenate(lists)
        real = allu[allu[:, 0] >= 0]
        tx, ty = D.tile_grid(W, H)
        assert len(real) == V * tx * ty
        keys = {tuple(r) for r in real}
        assert len(keys) == len(real)                      # no duplicates
        counts = [int((x[:, 0] >= 0).sum()) for x in lists]
        assert max(counts) - min(counts) <= 1              # balanced


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


def test_ipc_handle_bytes():
    """torch's shareable handle -> the raw 64-byte cudaIpcMemHandle_t."""
    import pytest
    raw = bytes(range(64))
    assert D.ipc_handle_bytes(raw) == raw
    assert D.ipc_handle_bytes(b"\x01c" + raw) == raw
    with pytest.raises(RuntimeError):
        D.ipc_handle_bytes(b"\x01e" + raw)
    with pytest.raises(RuntimeError):
        D.ipc_handle_bytes(raw[:10])
