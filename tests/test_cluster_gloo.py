"""Multi-process host logic of the cluster step on CPU (gloo, world_size 2 and 4):
replica-group payload exchange in member order, shard/replica group construction,
reduce-scatter geometry.  Payloads are produced and merged by the FP64 oracle, so the
check is exact: what the exchange hands to the merge equals what every member sent."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle.oracle import DEMO, FP16, FP32, RANDOM, TERNARY, Rep, restatement


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _body_arrays(rep, step, shard, n, seed):
    o = restatement()
    v = o.random_vector(seed, n)
    e = o.select_and_encode(v, rep, step, shard)
    wire = o.serialize(rep.scheme, e["freq_indices"], e["values"], rep.transfer_dtype)
    return e, np.frombuffer(wire[9:], np.uint8)


def _parse_body(body, rep, nvals):
    """the body layout of replicate.cpp:316-356 (indices then packed values)"""
    off = 0
    idx = None
    if rep.scheme == DEMO:
        idx = np.frombuffer(body[: 4 * nvals].tobytes(), np.uint32)
        off = 4 * nvals
    raw = body[off:]
    if rep.transfer_dtype == FP32:
        vals = np.frombuffer(raw[: 4 * nvals].tobytes(), np.float32).astype(np.float64)
    elif rep.transfer_dtype == FP16:
        vals = np.frombuffer(raw[: 2 * nvals].tobytes(), np.float16).astype(np.float64)
    else:
        codes = np.array([(raw[i // 4] >> (2 * (i % 4))) & 3 for i in range(nvals)])
        vals = np.where(codes == 1, 1.0, np.where(codes == 2, -1.0, 0.0))
    return idx, vals


def _exchange_worker(rank, world, port, cfgs, results):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2502_06728_b200.cluster import ReplicaExchange

    out = []
    for (scheme, dtype, sign, n) in cfgs:
        rep = Rep(scheme=scheme, chunk_size=64, top_k=8, compression=0.25, sign_mode=sign, transfer_dtype=dtype,
                  seed=77)
        e, body = _body_arrays(rep, 3, 0, n, 1000 + rank)
        cap = len(body) + 16
        own = torch.zeros(cap, dtype=torch.uint8)
        own[: len(body)] = torch.from_numpy(body.copy())
        ex = ReplicaExchange(dist.group.WORLD, world, cap, "cpu")
        bodies = ex.gather(own)
        parsed = [_parse_body(b.numpy(), rep, len(e["values"])) for b in bodies]
        o = restatement()
        q = o.decode_and_merge(rep, [p[1] for p in parsed], [p[0] for p in parsed], n, 3, 0)
        # what every member sent, recomputed locally from the known seeds
        sent = [_body_arrays(rep, 3, 0, n, 1000 + r)[0] for r in range(world)]
        wire_vals = [s["values"].astype(np.float32).astype(np.float64) if dtype == FP32 else s["values"] for s in sent]
        want = o.decode_and_merge(rep, wire_vals, [s["freq_indices"] for s in sent], n, 3, 0)
        out.append(bool(np.array_equal(q, want)))
    results[rank] = out
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_replica_exchange_member_order(world):
    cfgs = [(DEMO, FP32, True, 1000), (DEMO, FP16, False, 640), (RANDOM, FP32, False, 999), (DEMO, TERNARY, True, 333)]
    mgr = mp.Manager()
    results = mgr.dict()
    port = _free_port()
    mp.spawn(_exchange_worker, args=(world, port, cfgs, results), nprocs=world, join=True)
    for r in range(world):
        assert all(results[r]), (r, results[r])


def _groups_worker(rank, world, port, results):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2502_06728_b200.cluster import Topology, groups_for, reduce_scatter_mean, shard_spec

    topo = Topology(nodes=2, accels_per_node=2)
    sg, rg = groups_for(topo, rank)
    node, accel = divmod(rank, 2)
    # reduce-scatter inside the node: member-order mean then contiguous split (cluster.cpp:63-91)
    o = restatement()
    n = 2 * 257
    full = torch.from_numpy(o.random_vector(50 + rank, n).astype(np.float32))
    out = torch.empty(n // 2)
    reduce_scatter_mean(out, full, 2, sg)
    members = [o.random_vector(50 + node * 2 + a, n).astype(np.float32).astype(np.float64) for a in range(2)]
    want = o.grad_reduce_scatter(members)[accel]
    ok_rs = bool(np.allclose(out.numpy(), want, rtol=0, atol=1e-6))
    # replica group = same accel on every node, ordered by node
    t = torch.tensor([rank], dtype=torch.int64)
    got = [torch.zeros(1, dtype=torch.int64) for _ in range(2)]
    dist.all_gather(got, t, group=rg)
    ok_rg = [int(x) for x in got] == [0 * 2 + accel, 1 * 2 + accel]
    spec = shard_spec(213, 2, accel)
    ok_spec = (spec.offset, spec.extent, spec.real_len) == ((0, 107, 107) if accel == 0 else (107, 107, 106))
    results[rank] = (ok_rs, ok_rg, ok_spec)
    dist.destroy_process_group()


def test_hybrid_groups_and_reduce_scatter():
    """2 nodes x 2 accelerators: shard groups, replica groups, geometry (test_cluster.cpp:148-175)"""
    mgr = mp.Manager()
    results = mgr.dict()
    mp.spawn(_groups_worker, args=(4, _free_port(), results), nprocs=4, join=True)
    for r in range(4):
        assert results[r] == (True, True, True), (r, results[r])


def _bucket_exchange_worker(rank, world, port, results):
    """CollectiveExchange (the cluster's bucketed exchange): every bucket's bodies arrive in
    member order, whatever order the gathers complete in, and the agreement max-reduces the
    refusal flags over the world."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2502_06728_b200.cluster import CollectiveExchange

    ex = CollectiveExchange(None, dist.group.WORLD, None, members=world, shard_members=1)
    xfers = [48, 16, 112]
    ex.setup(xfers, "cpu")
    ex.begin_step()
    handles = []
    for bi, x in enumerate(xfers):
        ex.own(bi).copy_(torch.arange(x, dtype=torch.int64).to(torch.uint8) ^ (17 * rank + bi))
        handles.append(ex.start(bi))
    ok = True
    for bi in reversed(range(len(xfers))):  # merges may consume buckets in any order
        ptrs = ex.bodies(bi, handles[bi])
        base = ex.gathered[bi].data_ptr()
        for r in range(world):
            x = xfers[bi]
            ok &= ptrs[r] == base + r * x
            want = torch.arange(x, dtype=torch.int64).to(torch.uint8) ^ (17 * r + bi)
            ok &= bool(torch.equal(ex.gathered[bi][r * x:(r + 1) * x], want))
    flag = torch.tensor([1 if rank == world - 1 else 0], dtype=torch.int32)
    ex.agree(flag)
    results[rank] = (bool(ok), int(flag.item()))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_bucketed_exchange_and_agreement(world):
    mgr = mp.Manager()
    results = mgr.dict()
    mp.spawn(_bucket_exchange_worker, args=(world, _free_port(), results), nprocs=world, join=True)
    for r in range(world):
        assert results[r] == (True, 1), (r, results[r])
