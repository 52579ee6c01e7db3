"""One process per GPU: the reference's hybrid-sharded cluster step on real devices.

Mirrors VirtualCluster::run_step_hybrid (cluster.cpp:171-232) and the shard geometry of
VirtualCluster (cluster.cpp:101-158), with the simulated collectives replaced by
torch.distributed (NCCL over NVLink / NVSwitch on a B200 box, gloo on CPU for tests):

  world = nodes x accels_per_node, rank = node * A + accel        (cluster.hpp:81-90)
  shard group   {node * A + a : a}      -> gradient reduce-scatter (mean, contiguous split,
                                           cluster.cpp:63-91)
  replica group {n * A + accel : n}     -> all-gather of the fixed-size payloads, then a
                                           rank-ordered merge on every member
                                           (cluster.cpp:193-231, replicate.cpp:239-314)

The payload of a rank is exactly the reference's serialized body (indices then values
packed per transfer dtype, replicate.cpp:316-356), so the bytes NCCL moves per rank are
the reference's wire_bytes; `ledger` records them the way TrafficLedger does
(cluster.cpp:16-61): intra = reduce-scatter ring bytes, inter = bytes * (R - 1).
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field
from typing import Callable, List, Optional

import torch
import torch.distributed as dist

from . import _capi
from .core import (OptimizerConfig, OptimizerKind, ReplicatorConfig, Scheme, TransferDtype, _check, _ptr,
                   _stream,
                   context, status)
from ._capi import lib


@dataclass
class Topology:
    """ClusterTopology, cluster.hpp:15-21 (hybrid_sharded layout)."""
    nodes: int = 1
    accels_per_node: int = 1

    @property
    def world_size(self) -> int:
        return self.nodes * self.accels_per_node


@dataclass
class ShardSpec:
    """cluster.hpp:67-71"""
    offset: int
    extent: int
    real_len: int


def shard_spec(param_count: int, shards: int, shard_id: int) -> ShardSpec:
    """VirtualCluster ctor padding + ::shard (cluster.cpp:109-119, :148-158)."""
    padded = param_count + ((shards - param_count % shards) % shards)
    extent = padded // shards
    offset = shard_id * extent
    real = 0 if offset >= param_count else min(extent, param_count - offset)
    return ShardSpec(offset, extent, real)


@dataclass
class StepTraffic:
    """StepTraffic, cluster.hpp:31-39 (bytes only; time is measured, not modelled)."""
    step: int = 0
    intra_bytes: int = 0
    inter_bytes: int = 0
    reduce_scatter_events: int = 0
    synchronize_events: int = 0
    inter_bytes_reference: int = 0  # the reference wire format's bytes for the same exchange


def groups_for(topo: Topology, rank: int, backend: Optional[str] = None):
    """Build (shard_group, replica_group) for this rank; every rank must call this
    collectively with the same topology (dist.new_group is collective)."""
    A, N = topo.accels_per_node, topo.nodes
    shard_groups = [dist.new_group([n * A + a for a in range(A)], backend=backend) for n in range(N)]
    replica_groups = [dist.new_group([n * A + a for n in range(N)], backend=backend) for a in range(A)]
    node, accel = divmod(rank, A)
    return shard_groups[node], replica_groups[accel]


def reduce_scatter_mean(out: torch.Tensor, full: torch.Tensor, members: int, group) -> torch.Tensor:
    """grad_reduce_scatter (cluster.cpp:63-91): member mean, contiguous split.  NCCL
    averages in-network (ReduceOp.AVG, NVLS when available); gloo sums, then divides."""
    if members == 1:
        out.copy_(full[: out.numel()])
        return out
    if dist.get_backend(group) == "nccl":
        dist.reduce_scatter_tensor(out, full, op=dist.ReduceOp.AVG, group=group)
    else:
        dist.reduce_scatter_tensor(out, full, op=dist.ReduceOp.SUM, group=group)
        out.div_(members)
    return out


class ReplicaExchange:
    """All-gather of fixed-size payload bodies inside a replica group, in member order.

    Every member's body has the same size (the payload geometry depends only on the
    config, the step and the shard length, replicate.hpp:68-70), so one
    all_gather_into_tensor of `capacity` bytes per member moves exactly the bodies.
    """

    def __init__(self, group, members: int, capacity: int, device):
        self.group = group
        self.members = members
        self.capacity = capacity
        self.gathered = torch.empty(members * capacity, dtype=torch.uint8, device=device)

    def gather(self, own_body: torch.Tensor) -> List[torch.Tensor]:
        if self.members == 1:
            return [own_body[: self.capacity]]
        dist.all_gather_into_tensor(self.gathered, own_body[: self.capacity], group=self.group)
        return [self.gathered[r * self.capacity:(r + 1) * self.capacity] for r in range(self.members)]


class HybridCluster:
    """This rank's part of a FlexDeMo cluster step (cluster.cpp:171-232).

    Holds the rank's parameter shard and optimizer state on its GPU; `step()` takes the
    rank's full (padded) gradient, reduce-scatters it inside the node, runs the prepare
    kernel, all-gathers the payloads across the replica group and applies the merged
    update with the fused merge + apply kernel.
    """

    def __init__(self, topo: Topology, param_count: int, opt: OptimizerConfig, rep: ReplicatorConfig,
                 initial_params: torch.Tensor, rank: int, shard_group=None, replica_group=None,
                 buckets: int = 8, wire: str = "mask"):
        self.topo, self.opt, self.rep = topo, opt, rep
        self.rank = rank
        self.node, self.accel = divmod(rank, topo.accels_per_node)
        self.param_count = param_count
        self.spec = shard_spec(param_count, topo.accels_per_node, self.accel)
        self.device = initial_params.device
        self.shard_group, self.replica_group = shard_group, replica_group
        L = self.spec.real_len
        self.params = initial_params[self.spec.offset:self.spec.offset + L].clone().contiguous()
        if opt.kind == OptimizerKind.DemoSgd:
            self.m = torch.zeros(L, dtype=torch.float32, device=self.device)
        else:
            self.exp_avg = torch.zeros(L, dtype=torch.float32, device=self.device)
            self.exp_avg_sq = torch.zeros(L, dtype=torch.float32, device=self.device)
        self.steps = C.c_uint64(0)
        c = rep.c()
        self.capacity = int(lib.dmb_update_capacity(C.byref(c), L))
        self.own = torch.empty(self.capacity, dtype=torch.uint8, device=self.device)
        self.exchange = ReplicaExchange(replica_group, topo.nodes, self.capacity, self.device)
        self.shard_grad = torch.empty(self.spec.extent, dtype=torch.float32, device=self.device)
        self.ledger: List[StepTraffic] = []
        # Bucketed exchange (DeMo, R > 1): chunk-aligned slices of the shard, each prepared,
        # all-gathered and merged on its own, so the NVLink transfer of bucket b overlaps the
        # prepare of b+1 and the merge of b-1.  DeMo's selection is chunk-local, so every
        # bucket's payload is the reference's body of that sub-vector and the merged result
        # is the unbucketed one (Random / Striding / DiLoCo / Full use one bucket).
        # MASK exchange layout (include/demo_b200.h): u64 frequency mask per chunk + values,
        # lossless, used where the tensor-core AdamW kernels run (s = 64, whole chunks)
        self.mask_wire = (wire == "mask" and rep.scheme == Scheme.DeMo and opt.kind == OptimizerKind.DecoupledAdamW
                          and rep.chunk_size == 64 and L % 64 == 0)
        self.buckets = []
        if rep.scheme == Scheme.DeMo and topo.nodes > 1 and buckets > 1 and L > 0:
            tile = 128 * rep.chunk_size
            edges = sorted({min(L, (L * b // buckets) // tile * tile) for b in range(buckets)} | {L})
            vbits = 2 if (rep.sign_mode or rep.transfer_dtype == TransferDtype.Ternary) else \
                (16 if rep.transfer_dtype == TransferDtype.Fp16 else 32)
            for lo, hi in zip(edges[:-1], edges[1:]):
                cap = int(lib.dmb_update_capacity(C.byref(c), hi - lo))
                nch = (hi - lo) // 64
                body = 24 * nch if vbits == 2 else 8 * nch + (nch * rep.top_k * vbits + 7) // 8  # MASK(_SIGN)
                xfer = cap if not self.mask_wire else ((body + 15) // 16) * 16
                self.buckets.append(dict(lo=lo, hi=hi, cap=cap, xfer=xfer,
                                         own=torch.empty(cap, dtype=torch.uint8, device=self.device),
                                         gathered=torch.empty(topo.nodes * xfer, dtype=torch.uint8,
                                                              device=self.device)))
            self.payload_bytes_per_param = sum(b["xfer"] for b in self.buckets) / L
        self.ce = self._setup_ce_gather() if self.buckets else None

    def _reduce_scatter(self, grad_full: torch.Tensor) -> torch.Tensor:
        A = self.topo.accels_per_node
        if A == 1:
            return grad_full[: self.spec.extent]
        return reduce_scatter_mean(self.shard_grad, grad_full, A, self.shard_group)

    def _setup_ce_gather(self):
        """Copy-engine all-gather over symmetric memory: every member's bucket bodies live in
        a buffer mapped into all replica-group members; after a device-side barrier each
        member pulls the others' bodies with cudaMemcpyAsync (copy engines, no SMs), so the
        exchange overlaps the persistent step kernels.  Two buffers alternate between steps,
        so a member's next prepare never overwrites a body a peer is still copying.  Falls
        back to the NCCL all-gather when symmetric memory is unavailable."""
        if (self.topo.nodes < 2 or os.environ.get("DMB_CE_GATHER", "1") == "0"
                or dist.get_backend(self.replica_group) != "nccl"):
            return None
        try:
            import torch.distributed._symmetric_memory as symm

            offs, total = [], 0
            for b in self.buckets:
                offs.append(total)
                total += b["xfer"]
            bufs = [symm.empty(total, dtype=torch.uint8, device=self.device) for _ in range(2)]
            hdls = [symm.rendezvous(x, self.replica_group) for x in bufs]
            if hdls[0].world_size != self.topo.nodes or hdls[0].rank != self.node:
                return None
            return dict(bufs=bufs, hdls=hdls, offs=offs, stream=torch.cuda.Stream(self.device), step=0)
        except Exception:  # no symmetric-memory support here: NCCL all-gather
            return None

    def _step_bucketed(self, step: int, lr: float, g_shard: torch.Tensor, tr: StepTraffic) -> None:
        R = self.topo.nodes
        ctx = context(self.device).h
        c, o = self.rep.c(), self.opt.c()
        st = _stream(g_shard)
        sgd = self.opt.kind == OptimizerKind.DemoSgd
        pending = []

        def merge(b, hdr, work):
            own_ptr = None
            if isinstance(work, tuple):  # copy-engine gather: (done event, own body)
                torch.cuda.current_stream(self.device).wait_event(work[0])
                own_ptr = work[1].data_ptr()
            else:
                work.wait()  # the compute stream waits for the gather; the host does not
            lo, hi = b["lo"], b["hi"]
            ups = (_capi.Update * R)()
            for r in range(R):
                ups[r] = hdr
                ups[r].body = own_ptr if (own_ptr is not None and r == self.node) else \
                    b["gathered"][r * b["xfer"]:].data_ptr()
            if sgd:
                _check(lib.dmb_merge_apply_sgd(ctx, ups, R, C.byref(c), _ptr(self.params[lo:hi]),
                                               _ptr(g_shard[lo:hi]), hi - lo, step, float(lr), st))
            else:
                _check(lib.dmb_merge_apply_adamw(ctx, ups, R, self.node, C.byref(c), _ptr(self.params[lo:hi]),
                                                 _ptr(self.exp_avg[lo:hi]), _ptr(self.exp_avg_sq[lo:hi]),
                                                 C.byref(self.steps_b), _ptr(g_shard[lo:hi]), hi - lo, step,
                                                 C.byref(o), float(lr), st))

        steps0 = self.steps.value
        if self.mask_wire:
            _check(lib.dmb_set_wire_format(ctx, 1))
        try:
            self._pipeline(step, lr, g_shard, tr, merge, pending, steps0, ctx, c, o, st, sgd, R)
        finally:
            if self.mask_wire:
                lib.dmb_set_wire_format(ctx, 0)

    def _pipeline(self, step, lr, g_shard, tr, merge, pending, steps0, ctx, c, o, st, sgd, R):
        ce = self.ce
        if ce is not None:
            par = ce["step"] & 1
            ce["step"] += 1
            cbuf, hdl, cs = ce["bufs"][par], ce["hdls"][par], ce["stream"]
        for bi, b in enumerate(self.buckets):
            lo, hi = b["lo"], b["hi"]
            hdr = _capi.Update()
            own = cbuf[ce["offs"][bi]: ce["offs"][bi] + b["xfer"]] if ce is not None else b["own"]
            hdr.body = own.data_ptr()
            if sgd:
                _check(lib.dmb_demo_sgd_prepare(ctx, _ptr(g_shard[lo:hi]), _ptr(self.m[lo:hi]), _ptr(self.m[lo:hi]),
                                                hi - lo, C.byref(o), C.byref(c), step, self.accel, C.byref(hdr),
                                                None, None, st))
            else:
                _check(lib.dmb_adamw_prepare(ctx, _ptr(g_shard[lo:hi]), hi - lo, C.byref(c), step, self.accel,
                                             C.byref(hdr), None, st))
            tr.inter_bytes += int(hdr.bytes) * (R - 1)
            tr.inter_bytes_reference += int(lib.dmb_wire_bytes(hdr.n_values, hdr.n_indices,
                                                                self.rep.transfer_dtype)) * (R - 1)
            if ce is not None:
                ready = torch.cuda.Event()
                ready.record(torch.cuda.current_stream(self.device))
                cs.wait_event(ready)
                with torch.cuda.stream(cs):
                    hdl.barrier(channel=0)  # every member's prepare of this bucket is done
                    for r in range(R):
                        if r != self.node:
                            b["gathered"][r * b["xfer"]:(r + 1) * b["xfer"]].copy_(
                                hdl.get_buffer(r, (b["xfer"],), torch.uint8, ce["offs"][bi]), non_blocking=True)
                    done = torch.cuda.Event()
                    done.record(cs)
                work = (done, own)
            else:
                work = dist.all_gather_into_tensor(b["gathered"], b["own"][: b["xfer"]], group=self.replica_group,
                                                   async_op=True)
            if pending:
                self.steps_b = C.c_uint64(steps0)
                merge(*pending.pop())
            pending.append((b, hdr, work))
        self.steps_b = C.c_uint64(steps0)
        merge(*pending.pop())
        self.steps = self.steps_b  # every bucket advanced the AdamW counter from the same value

    def step(self, step: int, lr: float, grad_full: torch.Tensor, check: bool = True) -> StepTraffic:
        topo = self.topo
        L = self.spec.real_len
        tr = StepTraffic(step=step)
        g_shard = self._reduce_scatter(grad_full)[:L]  # the pad tail never leaves the node (:201)
        A = topo.accels_per_node
        tr.intra_bytes = A * (A - 1) * self.spec.extent * 4  # ring model, cluster.cpp:87
        tr.reduce_scatter_events = 1
        if self.buckets:
            tr.synchronize_events = 1
            self._step_bucketed(step, lr, g_shard, tr)
            if check:
                status(self.device)
            self.ledger.append(tr)
            return tr
        ctx = context(self.device).h
        st = _stream(g_shard)
        c, o = self.rep.c(), self.opt.c()
        hdr = _capi.Update()
        hdr.body = self.own.data_ptr()
        if self.opt.kind == OptimizerKind.DemoSgd:
            _check(lib.dmb_demo_sgd_prepare(ctx, _ptr(g_shard), _ptr(self.m), _ptr(self.m), L, C.byref(o),
                                            C.byref(c), step, self.accel, C.byref(hdr), None, None, st))
        else:
            _check(lib.dmb_adamw_prepare(ctx, _ptr(g_shard), L, C.byref(c), step, self.accel, C.byref(hdr),
                                         None, st))
        tr.inter_bytes = int(hdr.bytes) * (topo.nodes - 1)  # cluster.cpp:212
        tr.synchronize_events = 1
        R = topo.nodes
        ups = (_capi.Update * R)()
        if not hdr.empty:
            bodies = self.exchange.gather(self.own)
            for r in range(R):
                ups[r] = hdr
                ups[r].body = bodies[r].data_ptr()
        n_up = 0 if hdr.empty else R
        if self.opt.kind == OptimizerKind.DemoSgd:
            _check(lib.dmb_merge_apply_sgd(ctx, ups if n_up else None, n_up, C.byref(c), _ptr(self.params),
                                           _ptr(g_shard), L, step, float(lr), st))
        else:
            _check(lib.dmb_merge_apply_adamw(ctx, ups if n_up else None, n_up, self.node, C.byref(c),
                                             _ptr(self.params), _ptr(self.exp_avg), _ptr(self.exp_avg_sq),
                                             C.byref(self.steps), _ptr(g_shard), L, step, C.byref(o), float(lr),
                                             st))
        if check:
            status(self.device)
        self.ledger.append(tr)
        return tr
