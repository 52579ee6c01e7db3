#!/usr/bin/env python3
"""The shard-group reduce-scatter on its own, one process per GPU: NCCL reduce_scatter(AVG)
against dmb_grad_mean_pull reading the members' gradients from symmetric memory over NVLink, at a
few CTA budgets.  CUDA events on the launching stream, max over ranks; rank 0 prints JSON lines.

  python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1 tools/mgpu_pull_bench.py
"""
from __future__ import annotations

import ctypes as C
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", rank)))
    dev = torch.device("cuda", torch.cuda.current_device())
    dist.init_process_group("nccl", device_id=dev)
    import torch.distributed._symmetric_memory as symm

    from paper_2502_06728_b200._capi import lib
    from paper_2502_06728_b200.core import _check, context

    L = int(os.environ.get("PULL_PARAMS", 1_484_916_736))
    L -= L % (4 * world)
    ext = L // world
    buf = symm.empty(L, dtype=torch.float32, device=dev)
    hdl = symm.rendezvous(buf, dist.group.WORLD)
    buf.normal_(0, 1e-3)
    bases = [hdl.get_buffer(a, (L,), torch.float32, 0).data_ptr() for a in range(world)]
    out = torch.empty(ext, device=dev)
    ctx = context(dev).h
    st = torch.cuda.current_stream()
    sp = C.c_void_p(st.cuda_stream)

    def timed(fn, n=5):
        fn()
        torch.cuda.synchronize()
        dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        for _ in range(n):
            fn()
        e1.record(st)
        torch.cuda.synchronize()
        t = torch.tensor([e0.elapsed_time(e1) / n], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    res = []
    ms = timed(lambda: dist.reduce_scatter_tensor(out, buf, op=dist.ReduceOp.AVG))
    res.append({"what": "nccl reduce_scatter AVG", "ms": ms, "remote_GBps": (world - 1) * ext * 4 / ms / 1e6})
    for ctas in (8, 16, 20, 32, 64, 148):
        def pull():
            hdl.barrier(channel=0)
            ptrs = (C.c_void_p * world)(*[b + 4 * rank * ext for b in bases])
            _check(lib.dmb_grad_mean_pull(ctx, ptrs, world, ext, out.data_ptr(), ctas, sp))
        ms = timed(pull)
        res.append({"what": f"pull, {ctas} CTAs", "ms": ms, "remote_GBps": (world - 1) * ext * 4 / ms / 1e6})
    # the cluster's path: copy engines pull the peers' slices into local staging, then the local mean
    stage = {a: torch.empty(ext, device=dev) for a in range(world) if a != rank}
    views = [hdl.get_buffer(a, (L,), torch.float32, 0) for a in range(world)]
    for ctas in (16, 24, 32):
        def ce_pull():
            hdl.barrier(channel=0)
            for a, stg in stage.items():
                stg.copy_(views[a][rank * ext:(rank + 1) * ext], non_blocking=True)
            srcs = [buf[rank * ext:] if a == rank else stage[a] for a in range(world)]
            ptrs = (C.c_void_p * world)(*[t.data_ptr() for t in srcs])
            _check(lib.dmb_grad_mean_pull(ctx, ptrs, world, ext, out.data_ptr(), ctas, sp))
        ms = timed(ce_pull)
        res.append({"what": f"copy-engine pull + local mean, {ctas} CTAs", "ms": ms,
                    "remote_GBps": (world - 1) * ext * 4 / ms / 1e6})
    ms = timed(lambda: [stg.copy_(views[a][rank * ext:(rank + 1) * ext], non_blocking=True)
                        for a, stg in stage.items()])
    res.append({"what": "copy-engine pull alone", "ms": ms, "remote_GBps": (world - 1) * ext * 4 / ms / 1e6})
    if rank == 0:
        for r in res:
            print(json.dumps(dict(r, world=world, params=L)), flush=True)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
