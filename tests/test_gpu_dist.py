"""GPU tests of the multi-GPU direct-store path (dist.shared_image
/ render_direct): the render kernel stores a tile list's pixels at their image
positions (mfa_tiles.scatter), into a buffer rank 0 allocated and exported
with libmfa (mfa_ipc_alloc) and another process mapped (mfa_ipc_open on the
mapping rank's own device).  One GPU is
available, so the two-process test maps rank 0's image into rank 1 on the
same device (the same IPC and kernel path as across
NVLink; no kernel waits on another rank's kernel) with gloo for the handle
exchange and barriers; the result must equal the 1-GPU full-frame render bit
for bit."""
import os
import socket

import numpy as np
import pytest

from paper_2204_11762_b200 import dist as D, workloads as WL

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def _full(w, m):
    tf = torch.from_numpy(w.tf).cuda()
    img = m.render(w.cameras, tf, w.v_lo, w.v_hi, w.params)
    torch.cuda.synchronize()
    return img


def test_scatter_tiles_equal_full_frame():
    from paper_2204_11762_b200 import Model
    w = WL.make_config(2, width=200, height=120, n_views=2)
    m = Model.from_workload(w)
    full = _full(w, m)
    tf = torch.from_numpy(w.tf).cuda()
    img = torch.full_like(full, -1.0)
    for lst in D.assign_units(2, 200, 120, 3):   # three "ranks", padded lists
        m.render(w.cameras, tf, w.v_lo, w.v_hi, w.params, tiles=torch.from_numpy(lst).cuda(), out=img, scatter=True)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(img.cpu().numpy(), full.cpu().numpy())


def _worker(rank, world, port, out_path):
    import torch.distributed as dist
    from paper_2204_11762_b200 import Model
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    w = WL.make_config(2, width=160, height=96, n_views=2)
    m = Model.from_workload(w)
    tf = torch.from_numpy(w.tf).cuda()
    peer, err = D.shared_image((2, 96, 160, 4), torch.float32, rank)
    assert peer is not None, err
    if rank == 0:
        peer.fill_(-1.0)
        torch.cuda.synchronize()
    dist.barrier()

    def render_scatter(tiles, out):
        m.render(w.cameras, tf, w.v_lo, w.v_hi, w.params, tiles=tiles, out=out, scatter=True)

    img, n = D.render_direct(render_scatter, 2, 160, 96, rank, world, peer, device="cuda")
    assert n > 0
    if rank == 0:
        full = _full(w, m)
        np.save(out_path, np.stack([img.cpu().numpy(), full.cpu().numpy()]))
    dist.barrier()
    if rank != 0:
        peer.close()   # mfa_ipc_close
    dist.barrier()
    dist.destroy_process_group()


def test_two_process_ipc_direct_store(tmp_path):
    import torch.multiprocessing as mp
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    out = str(tmp_path / "img.npy")
    mp.start_processes(_worker, args=(2, port, out), nprocs=2, start_method="spawn", join=True)
    img, full = np.load(out)
    np.testing.assert_array_equal(img, full)


def test_bench_two_ranks_on_one_gpu(tmp_path):
    """`python bench.py --gpus 2` (no launcher) spawns two ranks itself; on a
    one-GPU box they share the device (gloo control plane, libmfa's IPC image
    for the pixels) and rank 0 prints one valid N = 2 line."""
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--gpus", "2", "--steps", "2", "--warmup", "1",
                        "--workload", "c2", "--views", "4", "--no-eval", "--no-cpu-baseline"],
                       capture_output=True, text=True, timeout=900, cwd=root)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [json.loads(x) for x in r.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1, r.stdout
    res = lines[0]
    assert res["n_gpus"] == 2 and res["steps"] == 2 and res["value"] > 0
    assert "views" in res["config"]["parallelism"]
    assert res["e2e"]["value"] > 0 and res["e2e"].get("host_image_ok", True)
