"""Multi-GPU screen-tile sharding (north_star "the control
points are replicated and the image is sharded by screen tiles, with an NCCL
gather of RGBA tiles over NVLink").

Every ray is independent given the replicated model (Algorithm 1 splits rows
over threads; "computation for all pixel values ... can also be
parallelized").  The work unit is a (view, 16x16 tile).

Assignment (assign_units, mode "auto"):
  * "views" when there are at least as many views as ranks (C5: 64 views):
    rank r renders views r, r+G, r+2G, ... (orbit angles spread over the
    whole circle, so the ranks' costs balance), each view whole and in the
    single-GPU supertile order -- a rank's kernel sees exactly the locality
    of the 1-GPU launch;
  * "rows" otherwise (one 2048^2 view of C4 on 8 GPUs): supertile rows
    (32-pixel bands, MFA_SUPERTILE = 2 tiles) dealt round-robin, each band
    in the 1-GPU supertile order;
  * "diagonal" (round 1, kept for the comparison in DESIGN.md §8): single
    tiles dealt along diagonals -- balanced to one tile, but a rank's tiles
    are G tiles apart, which destroys the neighbour-ray block reuse the
    render kernel lives on (measured by the 1-GPU rank emulation,
    bench.py --emulate).
Two ways to bring the pixels to rank 0:
  * "p2p" (default): rank 0's image is mapped into every rank through CUDA
    IPC and the render kernel stores each finished pixel straight to its
    position there (mfa_tiles.scatter = 1): the transfer is NVLink stores
    issued by the compute kernel itself, overlapped with the rest of the
    render -- no gather, no unpack (shared_image / render_direct).  The
    image is allocated by libmfa itself (mfa_ipc_alloc), so the export does
    not depend on the torch allocator; if any rank cannot map it the job
    falls back to NCCL;
  * "nccl": per view, a rank renders into a local buffer and a comm stream
    sends it to rank 0 (NCCL point-to-point over NVLink / NVSwitch) while the
    next view renders (ViewSender / gather_views_nccl); tile-sharded
    launches use one all_gather of packed tiles and rank 0's unpack kernel
    (render_sharded).
Per-pixel arithmetic does not depend on the assignment, so the G-GPU image
is bit-identical to the 1-GPU image.
"""
from __future__ import annotations

import numpy as np

TILE = 16


def tile_grid(width: int, height: int):
    return (width + TILE - 1) // TILE, (height + TILE - 1) // TILE


SUPERTILE = 2   # tiles per supertile edge (csrc/mfa_internal.cuh MFA_SUPERTILE)


def all_units(n_views: int, width: int, height: int) -> np.ndarray:
    """Every (view, tx, ty) unit in raster order, int32 (n, 3)."""
    tx, ty = tile_grid(width, height)
    v, y, x = np.meshgrid(np.arange(n_views), np.arange(ty), np.arange(tx), indexing="ij")
    return np.stack([v.ravel(), x.ravel(), y.ravel()], axis=1).astype(np.int32)


def supertile_order(views, width: int, height: int, rows=None) -> np.ndarray:
    """The (view, tx, ty) units of the given views (and supertile rows, or
    all) in the single-GPU kernel's full-frame order: view, supertile row,
    supertile column, tile inside the supertile (row-major)."""
    tx, ty = tile_grid(width, height)
    sty = (ty + SUPERTILE - 1) // SUPERTILE
    stx = (tx + SUPERTILE - 1) // SUPERTILE
    rows = np.arange(sty) if rows is None else np.asarray(list(rows), dtype=np.int64)
    views = np.asarray(list(views), dtype=np.int64)
    lt = np.arange(SUPERTILE * SUPERTILE)
    v, r, c, l = np.meshgrid(views, rows, np.arange(stx), lt, indexing="ij")
    x = c * SUPERTILE + l % SUPERTILE
    y = r * SUPERTILE + l // SUPERTILE
    keep = ((x < tx) & (y < ty)).ravel()
    u = np.stack([v.ravel(), x.ravel(), y.ravel()], axis=1)[keep]
    return np.ascontiguousarray(u, dtype=np.int32).reshape(-1, 3)


def pick_mode(n_views: int, world: int) -> str:
    return "views" if n_views >= world else "rows"


def rank_views(n_views: int, world: int, rank: int) -> list[int]:
    """Mode "views": the views rank renders (r, r+G, ...)."""
    return list(range(rank, n_views, world))


def _pad(lists):
    n = max((len(x) for x in lists), default=0)
    out = []
    for x in lists:
        pad = np.full((n - len(x), 3), -1, np.int32)
        out.append(np.ascontiguousarray(np.concatenate([x, pad])) if len(pad) else np.ascontiguousarray(x))
    return out


def assign_units(n_views: int, width: int, height: int, world: int, mode: str = "auto",
                 pad: bool = True) -> list[np.ndarray]:
    """Per-rank unit lists (int32 (n, 3) of (view, tx, ty)), each in the
    single-GPU supertile order; padded to equal length with view = -1
    entries (skipped by the render and unpack kernels) unless pad=False."""
    if mode == "auto":
        mode = pick_mode(n_views, world)
    tx, ty = tile_grid(width, height)
    if mode == "views":
        lists = [supertile_order(rank_views(n_views, world, r), width, height) for r in range(world)]
    elif mode == "rows":
        sty = (ty + SUPERTILE - 1) // SUPERTILE
        lists = [supertile_order(range(n_views), width, height, rows=range(r, sty, world)) for r in range(world)]
    elif mode == "diagonal":
        u = all_units(n_views, width, height)
        j = np.arange(len(u))
        row = j // tx
        col = j % tx
        # within tile-row r visit columns rotated by r, then deal round-robin
        order = np.lexsort(((col + row) % tx, row))
        owner = np.empty(len(u), np.int64)
        owner[order] = np.arange(len(u)) % world
        lists = [u[owner == r] for r in range(world)]
    else:
        raise ValueError(f"unknown assignment mode {mode!r}")
    lists = [np.ascontiguousarray(x, dtype=np.int32).reshape(-1, 3) for x in lists]
    return _pad(lists) if pad else lists


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


def render_direct(render_scatter, n_views, width, height, rank, world, peer_img, device=None, group=None):
    """Direct-store sharding: this rank renders its units straight into rank
    0's image (peer_img from shared_image).  render_scatter(tiles, out) launches
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


# ---------------------------------------------------------------------------
# the direct-store image: allocated by libmfa, mapped by every rank
# ---------------------------------------------------------------------------
def shared_image(shape, dtype, rank: int, group=None):
    """Rank 0 allocates the image with libmfa (mfa_ipc_alloc: cudaMalloc +
    cudaIpcGetMemHandle) and every other rank maps it on its own device
    (mfa_ipc_open).  Returns (image, ok): rank 0 a torch tensor, the others
    a _lib.PeerBuffer; ok is False on EVERY rank when any rank failed to
    allocate or map it (the caller then takes the NCCL path)."""
    import torch
    import torch.distributed as dist
    from ._lib import IpcBuffer, PeerBuffer
    elem = torch.finfo(dtype).bits // 8
    nbytes = int(np.prod(shape)) * elem
    img, meta, err = None, None, ""
    if rank == 0:
        try:
            buf = IpcBuffer(nbytes)
            img = buf.tensor(shape, dtype)
            meta = (buf.handle, 0, tuple(shape), str(dtype))
        except Exception as ex:   # allocation or export failed
            err = f"rank 0: {ex}"
    obj = [meta]
    dist.broadcast_object_list(obj, src=0, group=group)
    meta = obj[0]
    if rank != 0 and meta is not None:
        try:
            img = PeerBuffer(meta[0], meta[1], meta[2], dtype)
        except Exception as ex:
            err = f"rank {rank}: {ex}"
    status = [None] * dist.get_world_size(group)
    dist.all_gather_object(status, err, group=group)
    errs = [e for e in status if e]
    if errs or meta is None:
        if rank != 0 and img is not None:
            img.close()
        return None, "; ".join(errs) or "rank 0 could not export the image"
    return img, ""


# ---------------------------------------------------------------------------
# per-view NCCL gather overlapped with rendering (mode "views")
# ---------------------------------------------------------------------------
def gather_views_nccl(render_view, img0, n_views: int, rank: int, world: int, bufs=None, comm=None, group=None):
    """One step of the NCCL path for view-sharded launches (SURVEY §8(e):
    "gather view v on a comm stream while view v+1 renders").

    render_view(v, out) renders view v into out ([H,W,4]) on the current
    stream.  Rank 0 renders its own views straight into img0[v] and posts one
    receive per remote view into img0[v] (contiguous slices, no unpack);
    every other rank renders into two alternating local buffers (bufs) and
    sends each finished view from the comm stream, so the transfer of view v
    overlaps the render of the next.  Returns the list of outstanding works
    (the caller waits on them before using img0)."""
    import torch
    import torch.distributed as dist
    cuda = img0.is_cuda if img0 is not None else bufs[0].is_cuda
    cur = torch.cuda.current_stream() if cuda else None
    works = []
    if rank == 0:
        if cuda and comm is not None:
            comm.wait_stream(cur)
        ctx = torch.cuda.stream(comm) if (cuda and comm is not None) else _null()
        with ctx:
            for src in range(1, world):
                for v in rank_views(n_views, world, src):
                    works.append(dist.irecv(img0[v], src=src, group=group))
        for v in rank_views(n_views, world, 0):
            render_view(v, img0[v])
        return works
    pending = [None, None]
    for i, v in enumerate(rank_views(n_views, world, rank)):
        b = i & 1
        if pending[b] is not None:
            pending[b].wait()          # the compute stream waits until buffer b has been sent
        render_view(v, bufs[b])
        if cuda and comm is not None:
            comm.wait_stream(cur)      # the send starts after this view's render
            with torch.cuda.stream(comm):
                pending[b] = dist.isend(bufs[b], dst=0, group=group)
        else:
            pending[b] = dist.isend(bufs[b], dst=0, group=group)
        works.append(pending[b])
    return works


class _null:
    def __enter__(self):
        return self

    def __exit__(self, *a):
        return False
