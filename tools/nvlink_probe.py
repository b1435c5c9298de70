"""NVLink / NVSwitch probes for the multi-GPU numbers:
peer copy bandwidth between GPU pairs (copy engines, cudaMemcpyPeerAsync
via torch, one and both directions) and NCCL all-reduce bus bandwidth over
all visible GPUs (torch.distributed, one process per GPU).  CUDA events,
best of a few repetitions.

    python tools/nvlink_probe.py [MiB] > profiles/r2/nvlink_probe.json
"""
import json
import os
import socket
import sys

import torch


def _peer(nbytes, reps=5):
    out = []
    n = torch.cuda.device_count()
    for a, b in [(0, k) for k in range(1, n)]:
        x = torch.empty(nbytes, dtype=torch.uint8, device=f"cuda:{a}")
        y = torch.empty(nbytes, dtype=torch.uint8, device=f"cuda:{b}")
        x2 = torch.empty(nbytes, dtype=torch.uint8, device=f"cuda:{b}")
        y2 = torch.empty(nbytes, dtype=torch.uint8, device=f"cuda:{a}")
        y.copy_(x)
        torch.cuda.synchronize(a)
        torch.cuda.synchronize(b)
        best_uni, best_bi = 1e9, 1e9
        for _ in range(reps):
            with torch.cuda.device(a):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                y.copy_(x, non_blocking=True)
                e1.record()
                e1.synchronize()
                best_uni = min(best_uni, e0.elapsed_time(e1))
            # both directions at once: a -> b on a's stream, b -> a on b's stream
            sa, sb = torch.cuda.Stream(device=a), torch.cuda.Stream(device=b)
            torch.cuda.synchronize(a)
            torch.cuda.synchronize(b)
            with torch.cuda.device(a):
                f0 = torch.cuda.Event(enable_timing=True)
                f0.record(sa)
            with torch.cuda.stream(sa):
                y.copy_(x, non_blocking=True)
            with torch.cuda.stream(sb):
                y2.copy_(x2, non_blocking=True)
            with torch.cuda.device(b):
                gb = torch.cuda.Event()
                gb.record(sb)
            sa.wait_event(gb)
            with torch.cuda.device(a):
                f1 = torch.cuda.Event(enable_timing=True)
                f1.record(sa)
                f1.synchronize()
            best_bi = min(best_bi, f0.elapsed_time(f1))
        out.append({"pair": [a, b], "bytes": nbytes, "uni_GBps": nbytes / best_uni / 1e6,
                    "bidir_GBps_total": 2 * nbytes / best_bi / 1e6})
    return out


def _ar_worker(rank, world, port, nbytes, q):
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", rank=rank, world_size=world)
    t = torch.ones(nbytes // 4, dtype=torch.float32, device=f"cuda:{rank}")
    for _ in range(3):
        dist.all_reduce(t)
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(5):
        dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        dist.all_reduce(t)
        e1.record()
        e1.synchronize()
        best = min(best, e0.elapsed_time(e1))
    tt = torch.tensor([best], device=f"cuda:{rank}")
    dist.all_reduce(tt, op=dist.ReduceOp.MAX)
    if rank == 0:
        ms = float(tt.item())
        q.put({"ranks": world, "bytes": nbytes, "ms": ms, "algbw_GBps": nbytes / ms / 1e6,
               "busbw_GBps": 2 * (world - 1) / world * nbytes / ms / 1e6})
    dist.destroy_process_group()


def main():
    mib = int(sys.argv[1]) if len(sys.argv) > 1 else 256
    nbytes = mib << 20
    n = torch.cuda.device_count()
    res = {"gpus": n, "device": torch.cuda.get_device_name(0), "peer_copy": _peer(nbytes) if n > 1 else []}
    if n > 1:
        import torch.multiprocessing as mp

        s = socket.socket()
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
        s.close()
        ctx = mp.get_context("spawn")
        q = ctx.SimpleQueue()
        mp.spawn(_ar_worker, args=(n, port, nbytes, q), nprocs=n, join=True)
        res["nccl_allreduce"] = q.get()
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
