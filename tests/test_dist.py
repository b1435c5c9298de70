"""Multi-rank composite protocol on the CPU (gloo, world sizes 2 and 3).

Each rank owns a contiguous element range (synth.partition, the NekRS-style
split), agrees on the camera from the global bounds and on the colour range
from a global min/max, rasterises its own triangles into packed
depth|scalar keys, and the keys are min-reduced -- exactly the protocol
libnekb200 runs over NCCL (abi.cu run_step: range words appended to the key
buffer, one ncclMin reduce).  The composited image must equal the one-rank
image bit for bit, for any rank count (min is associative/commutative).
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import oracle as O
from paper_2312_09888_b200 import synth
from paper_2312_09888_b200.analysis import ortho_view

W, H = 96, 64
SURF = [("iso", "Q", 0.5), ("iso", "temperature", 0.6), ("slice", (0.3, 1.0, 0.2), 0.9)]
NEL = (4, 3, 3)
SIGN = np.uint64(1 << 63)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _rank_image(rank, size):
    E = NEL[0] * NEL[1] * NEL[2]
    e0, e1 = synth.partition(E, rank, size)
    c = synth.box(e0, e1, nel=NEL)
    lo = torch.tensor([c.x.min(), c.y.min(), c.z.min()], dtype=torch.float64)
    hi = torch.tensor([c.x.max(), c.y.max(), c.z.max()], dtype=torch.float64)
    dist.all_reduce(lo, op=dist.ReduceOp.MIN)
    dist.all_reduce(hi, op=dist.ReduceOp.MAX)
    bounds = (lo[0].item(), hi[0].item(), lo[1].item(), hi[1].item(), lo[2].item(), hi[2].item())
    view = ortho_view(bounds, W, H, 30.0, 40.0)
    cf = O.CaseFields(c.x, c.y, c.z, c.fields)
    tri, _, (cmin, cmax) = O.mc(cf, SURF, "temperature")
    keys = O.raster(tri, view, W, H)
    # gloo has no uint64 MIN: flip the sign bit so signed order == unsigned order
    t = torch.from_numpy((keys ^ SIGN).view(np.int64).copy())
    dist.all_reduce(t, op=dist.ReduceOp.MIN)
    rng = torch.tensor([cmin, -cmax], dtype=torch.float64)
    dist.all_reduce(rng, op=dist.ReduceOp.MIN)
    n = torch.tensor([len(tri)], dtype=torch.int64)
    dist.all_reduce(n)
    merged = t.numpy().view(np.uint64) ^ SIGN
    rgba, dep = O.resolve(merged, W, H, rng[0].item(), -rng[1].item())
    return rgba, dep, int(n.item())


def _worker(rank, size, port, out_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=size)
    try:
        rgba, dep, n = _rank_image(rank, size)
        if rank == 0:
            np.savez(os.path.join(out_dir, f"w{size}.npz"), rgba=rgba, dep=dep, n=n)
    finally:
        dist.destroy_process_group()


def _single():
    c = synth.box(nel=NEL)
    cf = O.CaseFields(c.x, c.y, c.z, c.fields)
    view = ortho_view((c.x.min(), c.x.max(), c.y.min(), c.y.max(), c.z.min(), c.z.max()), W, H, 30.0, 40.0)
    rgba, dep, n, _ = O.pipeline_mt(cf, SURF, "temperature", view, W, H, 1)
    return rgba, dep, n


@pytest.mark.parametrize("size", [2, 3])
def test_composite_is_rank_count_invariant(tmp_path, size):
    O.build()
    mp.spawn(_worker, args=(size, _free_port(), str(tmp_path)), nprocs=size, join=True)
    got = np.load(tmp_path / f"w{size}.npz")
    rgba, dep, n = _single()
    assert int(got["n"]) == n
    assert np.array_equal(got["rgba"], rgba)
    assert np.array_equal(got["dep"].view(np.uint32), dep.view(np.uint32))
    assert (rgba[..., 3] == 255).sum() > 500          # the image is not empty
