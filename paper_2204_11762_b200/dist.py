"""Multi-GPU screen-tile sharding (north_star "the control
points are replicated and the image is sharded by screen tiles, with an NCCL
gather of RGBA tiles over NVLink").

Every ray is independent given the replicated model (Algorithm 1 splits rows
over threads; "computation for all pixel values ... can also be
parallelized").  The work unit is a (view, 16x16 tile).  Units are
dealt round-robin to ranks along a diagonal order (each tile-row visited with
its columns rotated by the row index), so counts differ by at most one and
empty, cheap and ERT-heavy regions spread evenly.
Two ways to bring the pixels to rank 0:
  * "p2p" (default): rank 0's image is mapped into every rank through CUDA
    IPC and the render kernel stores each finished pixel straight to its
    position there (mfa_tiles.scatter = 1): the transfer is NVLink stores
    issued by the compute kernel itself, overlapped with the rest of the
    render -- no gather, no unpack (peer_image / render_direct);
  * "nccl": each rank renders into a packed tile buffer; one
    all_gather_into_tensor (NCCL over NVLink / NVSwitch) and rank 0's unpack
    kernel (render_sharded).
Per-pixel arithmetic does not depend on the assignment, so the G-GPU image
is bit-identical to the 1-GPU image.
"""
from __future__ import annotations

import numpy as np

TILE = 16


def tile_grid(width: int, height: int):
    return (width + TILE - 1) // TILE, (height + TILE - 1) // TILE


def all_units(n_views: int, width: int, height: int) -> np.ndarray:
    """Every (view, tx, ty) unit in raster order, int32 (n, 3)."""
    tx, ty = tile_grid(width, height)
    v, y, x = np.meshgrid(np.arange(n_views), np.arange(ty), np.arange(tx), indexing="ij")
    return np.stack([v.ravel(), x.ravel(), y.ravel()], axis=1).astype(np.int32)


def assign_units(n_views: int, width: int, height: int, world: int) -> list[np.ndarray]:
    """Per-rank unit lists, padded to equal length with view = -1 entries
    (skipped by the render and unpack kernels)."""
    u = all_units(n_views, width, height)
    tx, _ = tile_grid(width, height)
    j = np.arange(len(u))
    row = j // tx
    col = j % tx
    # within tile-row r visit columns rotated by r, then deal round-robin:
    # balanced to one unit, and a rank's tiles form diagonals, not columns
    order = np.lexsort(((col + row) % tx, row))
    owner = np.empty(len(u), np.int64)
    owner[order] = np.arange(len(u)) % world
    lists = [u[owner == r] for r in range(world)]
    n = max((len(x) for x in lists), default=0)
    out = []
    for x in lists:
        pad = np.full((n - len(x), 3), -1, np.int32)
        out.append(np.ascontiguousarray(np.concatenate([x, pad])) if len(pad) else np.ascontiguousarray(x))
    return out


def render_sharded(render_tiles, unpack, n_views, width, height, rank, world, device=None,
                   channels=4, dtype=None, group=None):
    """Render this rank's units, gather every rank's packed tiles, unpack on rank 0.

    render_tiles(tiles_int32_tensor) -> packed tensor [n, 16, 16, channels]
    unpack(packed_all, tiles_all) -> image (rank 0 only)
    Returns (image or None, n_local_units)."""
    import torch
    import torch.distributed as dist
    lists = assign_units(n_views, width, height, world)
    mine = torch.from_numpy(lists[rank])
    if device is not None:
        mine = mine.to(device)
    packed = render_tiles(mine)
    if world == 1:
        return unpack(packed, mine), len(lists[rank])
    gathered = torch.empty((world * packed.shape[0],) + tuple(packed.shape[1:]), dtype=packed.dtype,
                           device=packed.device)
    dist.all_gather_into_tensor(gathered, packed.contiguous(), group=group)
    if rank != 0:
        return None, len(lists[rank])
    tiles_all = torch.from_numpy(np.concatenate(lists)).to(packed.device)
    return unpack(gathered, tiles_all), len(lists[rank])


def ipc_handle_bytes(h: bytes) -> bytes:
    """The 64-byte cudaIpcMemHandle_t inside torch's shareable handle: raw
    (older torch) or prefixed by a version byte and the segment type 'c'
    (a cudaMalloc segment).  Expandable segments carry no cudaIpc handle."""
    if len(h) == 64:
        return h
    if len(h) == 66 and h[1:2] == b"c":
        return h[2:]
    raise RuntimeError(f"unsupported CUDA IPC handle from torch (length {len(h)}, type {h[1:2]!r}); "
                       "the direct-store path needs the default (non-expandable) CUDA allocator")


def peer_image(img, rank: int, group=None):
    """Rank 0's image on every rank: rank 0 gets img back, the others a
    _lib.PeerBuffer mapping it on their OWN device.

    Rank 0 exports the image's allocation (the CUDA IPC handle and the
    tensor's byte offset in it, from torch's storage sharing); every other
    rank maps it with mfa_ipc_open on its current device
    (cudaIpcMemLazyEnablePeerAccess), so its render kernel stores into rank
    0's HBM over NVLink -- or locally when both ranks share one device."""
    import torch.distributed as dist
    if rank == 0:
        st = img.untyped_storage()
        info = st._share_cuda_()          # (device, handle, size, offset in the allocation, ...)
        meta = (ipc_handle_bytes(bytes(info[1])), int(info[3]) + img.storage_offset() * img.element_size(),
                tuple(img.shape), str(img.dtype))
    obj = [meta if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0, group=group)
    if rank == 0:
        return img
    handle, offset, shape, dtype = obj[0]
    from ._lib import PeerBuffer
    return PeerBuffer(handle, offset, shape, dtype)


def render_direct(render_scatter, n_views, width, height, rank, world, peer_img, device=None, group=None):
    """Direct-store sharding: this rank renders its units straight into rank
    0's image (peer_img from peer_image).  render_scatter(tiles, out) launches
    the render with scatter = 1.  After the call every rank's stores are
    complete and visible to rank 0 (stream synchronisation + barrier)."""
    import torch
    import torch.distributed as dist
    lists = assign_units(n_views, width, height, world)
    mine = torch.from_numpy(lists[rank])
    if device is not None:
        mine = mine.to(device)
    render_scatter(mine, peer_img)
    torch.cuda.current_stream().synchronize()
    if world > 1:
        dist.barrier(group=group)
    return peer_img if rank == 0 else None, len(lists[rank])
