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

One step runs in three phases (`begin`, `agree`, `commit`; `step` runs all three):

  begin   reduce-scatter, then per bucket (chunk-aligned slices of the shard for DeMo, whose
          selection is chunk-local, so each bucket's payload is the reference's payload of
          that sub-vector): the prepare kernel, then the start of the bucket's exchange, which
          overlaps the prepares of the later buckets;
  agree   every prepare has latched a non-finite gradient it saw (require_finite,
          vec.cpp:7-16); the latches are max-reduced over the world on the device, so a bad
          gradient anywhere refuses the whole step everywhere, as the reference checks every
          gradient before any state changes (cluster.cpp:182);
  commit  per bucket: wait for its exchange, the fused merge + apply kernel (a no-op once
          the step is refused), then the status check.  Momentum (SGD) is double buffered
          and the host-side step counter restored, so a refused step leaves every state
          vector as it was (optim.cpp:21).

At R = 1 (S x 1 layouts) there is nothing to exchange and DeMo runs the fused one-pass step
kernel with double-buffered outputs, swapped when the step succeeds.

The shard group's reduce-scatter is NCCL's, or -- HybridCluster(pull_grads=True), gradients
written into grad_buffer(step) (symmetric memory) -- fused into the step kernels: the AdamW
prepare / one-pass step average the members' slices of the shard in their gradient load
(dmb_*_members; the peers' slices read over NVLink by the kernel's TMA for the one-pass step,
staged by the copy engines for the prepare), DeMo-SGD takes the mean as a CTA-budgeted pass of
its own (dmb_grad_mean_pull) beside the step kernels; every variant is bit-identical to NCCL's.

Environment switches (measurement and fallbacks; the defaults are the measured best):
  DMB_CE_GATHER=0      replica exchange by NCCL all-gather instead of copy engines
  DMB_GATHER_BUDGET=n  exchange memory budget in bytes (above it: memory-bounded windows)
  DMB_OVERLAP=1        overlapped merges on split SMs (DMB_MERGE_SMS: the merges' share)
  DMB_PULL_FUSED=0     pulled reduce-scatter as a mean pass even for AdamW
  DMB_PULL_STAGED=1    stage the peers' slices by copy engines for the one-pass step too
  DMB_CE_PEER_STREAMS=1  pull the peers' slices on one copy stream per peer (measured slower)

The exchange is injectable: `CollectiveExchange` (torch.distributed all-gather, any
backend), `CopyEngineExchange` (symmetric memory pulled by copy engines over NVLink, NCCL
only for the agreement), `LocalExchange` (R members in one process on one GPU, tests).  The
DeMo payload layout per bucket comes from the library before anything runs
(dmb_plan_exchange): the lossless MASK layout where the tensor-core encoders run, else the
reference body; every prepare's header is checked against that plan.  `ledger` records the
bytes the way TrafficLedger does (cluster.cpp:16-61): intra = reduce-scatter ring bytes,
inter = bytes * (R - 1), beside the reference wire format's bytes for the same exchange.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass
from typing import List, Optional

import torch
import torch.distributed as dist

from . import _capi
from ._capi import lib
from .core import (ConfigError, OptimizerConfig, OptimizerKind, ProtocolError, ReplicatorConfig, Scheme, StepTrace,
                   TrainingError,
                   _check, _ptr, _stream, context, status)


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


# ------------------------------------------------------------------ exchanges
class CollectiveExchange:
    """torch.distributed all-gather of each bucket's bodies in the replica group (NCCL over
    NVLink on the GPU box, gloo in the CPU tests); agreement by an all-reduce over `world`."""

    def __init__(self, shard_group, replica_group, world_group=None, members: int = 1, shard_members: int = 1):
        self.shard_group, self.replica_group, self.world_group = shard_group, replica_group, world_group
        self.members, self.shard_members = members, shard_members

    def setup(self, xfers: List[int], device) -> None:
        self.xfers = xfers
        self.own_slots = [torch.empty(x, dtype=torch.uint8, device=device) for x in xfers]
        self.gathered = [torch.empty(self.members * x, dtype=torch.uint8, device=device) if self.members > 1 else None
                         for x in xfers]

    def begin_step(self) -> None:
        pass

    def own(self, bi: int) -> torch.Tensor:
        return self.own_slots[bi]

    def reduce_scatter(self, out: torch.Tensor, full: torch.Tensor) -> torch.Tensor:
        return reduce_scatter_mean(out, full, self.shard_members, self.shard_group)

    def start(self, bi: int):
        if self.members == 1:
            return None
        return dist.all_gather_into_tensor(self.gathered[bi], self.own_slots[bi], group=self.replica_group,
                                           async_op=True)

    def bodies(self, bi: int, handle) -> List[int]:
        if self.members == 1:
            return [self.own_slots[bi].data_ptr()]
        handle.wait()  # the compute stream waits for the gather; the host does not (NCCL)
        x = self.xfers[bi]
        return [self.gathered[bi][r * x:].data_ptr() for r in range(self.members)]

    def agree(self, flag: torch.Tensor) -> None:
        if self.world_group is not None or dist.is_initialized():
            if dist.get_world_size(self.world_group) > 1:
                dist.all_reduce(flag, op=dist.ReduceOp.MAX, group=self.world_group)


class CopyEngineExchange(CollectiveExchange):
    """The bodies live in symmetric memory (one buffer mapped into every replica-group
    member, two alternating by step so a member's next prepare never overwrites a body a peer
    is still copying).  After a device-side barrier each member pulls the others' bodies with
    cudaMemcpyAsync -- copy engines over NVLink, no SMs -- on a side stream, so the exchange
    runs under the persistent prepare kernels of the later buckets."""

    def __init__(self, shard_group, replica_group, world_group, members: int, shard_members: int, node: int):
        super().__init__(shard_group, replica_group, world_group, members, shard_members)
        self.node = node

    def setup(self, xfers: List[int], device) -> None:
        import torch.distributed._symmetric_memory as symm

        self.xfers = xfers
        self.offs, total = [], 0
        for x in xfers:
            self.offs.append(total)
            total += x
        self.bufs = [symm.empty(total, dtype=torch.uint8, device=device) for _ in range(2)]
        self.hdls = [symm.rendezvous(b, self.replica_group) for b in self.bufs]
        if self.hdls[0].world_size != self.members or self.hdls[0].rank != self.node:
            raise RuntimeError("symmetric-memory rendezvous does not match the replica group")
        self.gathered = [torch.empty(self.members * x, dtype=torch.uint8, device=device) for x in xfers]
        self.stream = torch.cuda.Stream(device)
        self.device = device
        self.parity = 1

    def begin_step(self) -> None:
        self.parity ^= 1

    def own(self, bi: int) -> torch.Tensor:
        o = self.offs[bi]
        return self.bufs[self.parity][o:o + self.xfers[bi]]

    def start(self, bi: int):
        ready = torch.cuda.Event()
        ready.record(torch.cuda.current_stream(self.device))
        self.stream.wait_event(ready)
        hdl, x, o = self.hdls[self.parity], self.xfers[bi], self.offs[bi]
        with torch.cuda.stream(self.stream):
            hdl.barrier(channel=0)  # every member's prepare of this bucket is done
            for r in range(self.members):
                if r != self.node:
                    self.gathered[bi][r * x:(r + 1) * x].copy_(hdl.get_buffer(r, (x,), torch.uint8, o), non_blocking=True)
            done = torch.cuda.Event()
            done.record(self.stream)
        return done

    def bodies(self, bi: int, handle) -> List[int]:
        torch.cuda.current_stream(self.device).wait_event(handle)
        x = self.xfers[bi]
        return [self.own(bi).data_ptr() if r == self.node else self.gathered[bi][r * x:].data_ptr()
                for r in range(self.members)]


class LocalHub:
    """R x A members of one cluster in ONE process on one GPU (tests): the members' bodies
    are read in place, the reduce-scatter is the member-order mean (dmb_grad_mean), and the
    agreement is the max of the members' flags.  Drive the members phase by phase:
    hub.grads[rank] = ...; every member.begin(); hub.agree(); every member.commit()."""

    def __init__(self, topo: Topology):
        self.topo = topo
        self.members: dict = {}
        self.grads: dict = {}

    def agree(self) -> None:
        flags = [m.flag for m in self.members.values()]
        top = torch.stack(flags).max(dim=0).values
        for f in flags:
            f.copy_(top)


class LocalExchange(CollectiveExchange):
    def __init__(self, hub: LocalHub, rank: int):
        A = hub.topo.accels_per_node
        super().__init__(None, None, None, hub.topo.nodes, A)
        self.hub, self.rank = hub, rank
        self.node, self.accel = divmod(rank, A)

    def setup(self, xfers: List[int], device) -> None:
        self.xfers = xfers
        self.own_slots = [torch.empty(x, dtype=torch.uint8, device=device) for x in xfers]

    def reduce_scatter(self, out: torch.Tensor, full: torch.Tensor) -> torch.Tensor:
        A = self.shard_members
        if A == 1:
            out.copy_(full[: out.numel()])
            return out
        n = out.numel()
        ins = [self.hub.grads[self.node * A + a][self.accel * n:(self.accel + 1) * n] for a in range(A)]
        arr = (C.c_void_p * A)(*[g.data_ptr() for g in ins])
        _check(lib.dmb_grad_mean(context(out.device).h, arr, A, n, _ptr(out), _stream(out)))
        return out

    def start(self, bi: int):
        return None

    def bodies(self, bi: int, handle) -> List[int]:
        A = self.shard_members
        return [self.hub.members[n * A + self.accel].exchange.own_slots[bi].data_ptr() for n in range(self.members)]

    def agree(self, flag: torch.Tensor) -> None:
        pass  # the hub agrees for every member between the phases


# ------------------------------------------------------------------ the cluster step
class HybridCluster:
    """This rank's part of a FlexDeMo cluster step (cluster.cpp:171-232).

    Holds the rank's parameter shard and optimizer state on its GPU; `step()` takes the
    rank's full (padded) gradient, reduce-scatters it inside the node, prepares, exchanges
    the payloads across the replica group and applies the merged update (see the module
    docstring for the phases and the failure semantics).
    """

    def __init__(self, topo: Topology, param_count: int, opt: OptimizerConfig, rep: ReplicatorConfig,
                 initial_params: torch.Tensor, rank: int, shard_group=None, replica_group=None,
                 buckets: int = 8, wire: str = "mask", exchange=None, world_group=None, trace: bool = False,
                 pull_grads: bool = False, pull_ctas: int = 40, overlap: Optional[bool] = None,
                 merge_sms: int = 90):
        self.topo, self.opt, self.rep = topo, opt, rep
        self.rank = rank
        self.node, self.accel = divmod(rank, topo.accels_per_node)
        self.param_count = param_count
        self.spec = shard_spec(param_count, topo.accels_per_node, self.accel)
        self.device = initial_params.device
        R, A = topo.nodes, topo.accels_per_node
        L = self.spec.real_len
        self.sgd = opt.kind == OptimizerKind.DemoSgd
        # R = 1 DeMo: one pass, double-buffered outputs; a traced step (StepTrace of every SGD
        # prepare, optim.hpp:33-38) takes the prepare -> merge(R = 1) path instead
        self.fused = R == 1 and rep.scheme == Scheme.DeMo and L > 0 and not trace
        self._trace_bufs = (torch.empty(L, device=initial_params.device),
                            torch.empty(L, device=initial_params.device)) if trace and opt.kind == OptimizerKind.DemoSgd \
            else None
        self.params = initial_params[self.spec.offset:self.spec.offset + L].clone().contiguous()
        z = lambda: torch.zeros(L, dtype=torch.float32, device=self.device)  # noqa: E731
        if self.sgd:
            self.m, self._m_next = z(), z()
        else:
            self.exp_avg, self.exp_avg_sq = z(), z()
        if self.fused:  # the fused step writes p (and the moments) into spares, swapped on success
            self._p_next = z()
            if not self.sgd:
                self._ea_next, self._es_next = z(), z()
        self.steps = 0
        self.shard_grad = torch.empty(self.spec.extent, dtype=torch.float32, device=self.device)
        self.flag = torch.zeros(1, dtype=torch.int32, device=self.device)
        self.ledger: List[StepTraffic] = []
        ctx = context(self.device).h
        if wire not in ("mask", "reference"):
            raise ConfigError(f"unknown exchange layout {wire!r}")
        self.wire = wire
        # buckets: chunk-aligned slices of the shard (DeMo), one bucket for the other schemes
        # pulled reduce-scatter (A > 1): the members' full gradients live in symmetric memory and
        # every rank pulls its shard's slices over NVLink bucket by bucket, under the step kernels
        self.pull = bool(pull_grads) and A > 1 and shard_group is not None
        tile = 128 * max(rep.chunk_size, 1)
        nb = buckets if (rep.scheme == Scheme.DeMo and (R > 1 or self.pull)) else 1
        edges = sorted({min(L, (L * b // nb) // tile * tile) for b in range(nb)} | {L})
        self.buckets = [dict(lo=lo, hi=hi) for lo, hi in zip(edges[:-1], edges[1:])] if L else []
        # the payload layout of every bucket, from the library, before anything runs
        c = rep.c()
        lib.dmb_set_wire_format(ctx, 1 if wire == "mask" else 0)
        try:
            for b in self.buckets:
                h = _capi.Update()
                _check(lib.dmb_plan_exchange(ctx, C.byref(c), b["hi"] - b["lo"], 0, self.accel, C.byref(h)))
                b["format"] = int(h.wire_format)
                b["bytes"] = int(h.bytes)
                b["xfer"] = max(16, (int(lib.dmb_update_capacity(C.byref(c), b["hi"] - b["lo"])) if not h.wire_format
                                     else (int(h.bytes) + 15) // 16 * 16))
        finally:
            lib.dmb_set_wire_format(ctx, 0)
        self.mask_wire = any(b["format"] for b in self.buckets)
        self.payload_bytes_per_param = (sum(b["bytes"] for b in self.buckets) / L) if L else 0.0
        # memory: every bucket's own slot(s) and R gathered copies stay resident through a step;
        # above the budget (DMB_GATHER_BUDGET bytes, default a quarter of the device) the step runs
        # the buckets in windows that fit, after a finiteness pre-check of the whole shard that
        # the ranks agree on first (one extra read of the gradient), so a refused step still
        # changes nothing
        self.window = len(self.buckets)
        if R > 1 and self.buckets and not self.fused:
            budget = int(os.environ.get("DMB_GATHER_BUDGET", "0")) or int(
                0.25 * torch.cuda.get_device_properties(self.device).total_memory)
            per = (R + 2) * max(b["xfer"] for b in self.buckets)
            if per * len(self.buckets) > budget:
                self.window = max(1, budget // per)
        if exchange is None:
            exchange = self._default_exchange(shard_group, replica_group, world_group)
        if self.window < len(self.buckets):
            if isinstance(exchange, LocalExchange):
                raise ConfigError("the bucket windows of a memory-bounded step need a collective exchange")
            if isinstance(exchange, CopyEngineExchange):  # slots are reused within a step: stream-ordered NCCL
                exchange = CollectiveExchange(shard_group, replica_group, world_group, R, A)
        self.exchange = exchange
        if self.buckets and not self.fused:
            if self.window < len(self.buckets):
                mx = max(b["xfer"] for b in self.buckets)
                exchange.setup([mx] * self.window, self.device)
            else:
                exchange.setup([b["xfer"] for b in self.buckets], self.device)
        self.ce = exchange if isinstance(exchange, CopyEngineExchange) else None
        if isinstance(exchange, LocalExchange):
            exchange.hub.members[rank] = self
        if self.pull:
            self._setup_pull(shard_group, pull_ctas)
        # overlapped merges (opt-in: overlap=True or DMB_OVERLAP=1; R > 1, DeMo, one process per GPU):
        # the merge of bucket b runs on its own stream and its own SMs while the prepares of the
        # later buckets run on the rest -- the select-bound encode beside the HBM-bound merge --
        # writing into spare state buffers, so the step can merge before the ranks agree on it and
        # a refused step keeps the old state (bit-identical to the sequential step).  Measured on
        # B200 at 1 x 2 (OLMo-1B AdamW): 11.9 ms at the best split (90 merge SMs) against 11.3 ms
        # sequential, so it is off by default.  Needs the spares to fit (4 B/param SGD, 12 AdamW).
        spare = L * (4 if self.sgd else 12)
        auto = (R > 1 and rep.scheme == Scheme.DeMo and L > 0 and not self.fused and not self.pull and not trace
                and self.window == len(self.buckets) and not isinstance(exchange, LocalExchange)
                and torch.cuda.mem_get_info(self.device)[0] > spare + (8 << 30))
        if overlap is None and os.environ.get("DMB_OVERLAP"):
            overlap = os.environ["DMB_OVERLAP"] != "0"
        merge_sms = int(os.environ.get("DMB_MERGE_SMS", merge_sms))
        self.overlap = bool(overlap) and auto
        if self.overlap:
            self._p_next = z()
            if not self.sgd:
                self._ea_next, self._es_next = z(), z()
            self._mstream = torch.cuda.Stream(self.device)
            sms = torch.cuda.get_device_properties(self.device).multi_processor_count
            self._m_sms = max(1, min(int(merge_sms), sms - 1))
            self._e_sms = sms - self._m_sms

    def _default_exchange(self, shard_group, replica_group, world_group):
        R, A = self.topo.nodes, self.topo.accels_per_node
        if (R > 1 and os.environ.get("DMB_CE_GATHER", "1") != "0" and replica_group is not None
                and dist.get_backend(replica_group) == "nccl"):
            try:
                return CopyEngineExchange(shard_group, replica_group, world_group, R, A, self.node)
            except Exception:  # no symmetric-memory support: the NCCL all-gather
                pass
        return CollectiveExchange(shard_group, replica_group, world_group, R, A)

    # ---- phases -----------------------------------------------------------------
    def begin(self, step: int, lr: float, grad_full: torch.Tensor, trace=None) -> None:
        """reduce-scatter, every bucket's prepare and the start of its exchange; `trace`
        (SGD, a member built with trace=True) is called as trace(node, accel, StepTrace) with
        the shard's m_accum, local_q and m_after (device views) after the prepares, as
        run_step_hybrid's TraceSink (cluster.cpp:205-209)"""
        topo, L = self.topo, self.spec.real_len
        A, R = topo.accels_per_node, topo.nodes
        tr = StepTraffic(step=step, reduce_scatter_events=1, synchronize_events=1)
        tr.intra_bytes = A * (A - 1) * self.spec.extent * 4  # ring model, cluster.cpp:87
        self._tr, self._step, self._lr = tr, step, float(lr)
        self._steps0 = self.steps
        # the pad tail never leaves the node (cluster.cpp:201)
        pulled = self.pull and any(grad_full.data_ptr() == b.data_ptr() for b in self._gbufs)
        if pulled:
            self.g_shard = self.shard_grad[:L]
            self._pull_start(grad_full)
        else:
            self._pulled = None
            self.g_shard = grad_full[:L] if A == 1 else self.exchange.reduce_scatter(self.shard_grad, grad_full)[:L]
        self._pending = []
        if not L:
            return
        ctx = context(self.device).h
        st = _stream(self.g_shard)
        c, o = self.rep.c(), self.opt.c()
        if self.fused:
            try:
                self._fused(ctx, c, o, st)
            finally:
                if self._pulled:
                    lib.dmb_set_sm_reserve(0)
        elif self.window < len(self.buckets):
            self._windowed(ctx, c, o, st)
            return
        else:
            self.exchange.begin_step()
            lib.dmb_set_wire_format(ctx, 1 if self.wire == "mask" else 0)
            try:
                for bi, b in enumerate(self.buckets):
                    lo, hi = b["lo"], b["hi"]
                    self._pull_wait(bi)
                    hdr = _capi.Update()
                    hdr.body = self.exchange.own(bi).data_ptr()
                    tb = self._trace_bufs if trace is not None else None
                    if self.overlap:
                        lib.dmb_set_sm_reserve(self._m_sms)  # the prepares leave the merges their SMs
                    if self.sgd and self._pulled and self._pull_fused:  # the shard's mean fused into the prepare
                        srcs = self._members_at(lo)
                        _check(lib.dmb_demo_sgd_prepare_members(ctx, srcs, len(srcs), _ptr(self.g_shard[lo:hi]),
                                                                _ptr(self.m[lo:hi]), _ptr(self._m_next[lo:hi]),
                                                                hi - lo, C.byref(o), C.byref(c), step, self.accel,
                                                                C.byref(hdr), st))
                    elif self.sgd:
                        _check(lib.dmb_demo_sgd_prepare(ctx, _ptr(self.g_shard[lo:hi]), _ptr(self.m[lo:hi]),
                                                        _ptr(self._m_next[lo:hi]), hi - lo, C.byref(o), C.byref(c),
                                                        step, self.accel, C.byref(hdr),
                                                        _ptr(tb[0][lo:hi]) if tb else None,
                                                        _ptr(tb[1][lo:hi]) if tb else None, st))
                    elif self._pulled and self._pull_fused:  # the shard's mean fused into the prepare
                        srcs = self._members_at(lo)
                        _check(lib.dmb_adamw_prepare_members(ctx, srcs, len(srcs), _ptr(self.g_shard[lo:hi]),
                                                             hi - lo, C.byref(c), step, self.accel, C.byref(hdr),
                                                             st))
                    else:
                        _check(lib.dmb_adamw_prepare(ctx, _ptr(self.g_shard[lo:hi]), hi - lo, C.byref(c), step,
                                                     self.accel, C.byref(hdr), None, st))
                    if not hdr.empty and (int(hdr.wire_format) != b["format"] or int(hdr.bytes) > b["xfer"]):
                        raise ProtocolError(f"bucket {bi}: the prepare produced layout {hdr.wire_format} / "
                                            f"{hdr.bytes} B, planned {b['format']} / {b['xfer']} B")
                    tr.inter_bytes += int(hdr.bytes) * (R - 1)  # cluster.cpp:212
                    tr.inter_bytes_reference += int(lib.dmb_wire_bytes(hdr.n_values, hdr.n_indices,
                                                                        self.rep.transfer_dtype)) * (R - 1)
                    handle = self.exchange.start(bi) if not hdr.empty else None
                    self._pending.append((b, hdr, handle))
                    if self.overlap:
                        self._merge_to(ctx, c, o, bi, b, hdr, handle)
            finally:
                lib.dmb_set_wire_format(ctx, 0)
                if self._pulled or self.overlap:
                    lib.dmb_set_sm_reserve(0)
            if self.overlap:
                self._mdone = torch.cuda.Event()
                self._mdone.record(self._mstream)
            if trace is not None:
                if self._trace_bufs is None:
                    raise ConfigError("a traced step needs a DemoSgd member built with trace=True")
                trace(self.node, self.accel, StepTrace(m_accum=self._trace_bufs[1], local_q=self._trace_bufs[0],
                                                       m_after=self._m_next))
        _check(lib.dmb_latch_export(ctx, _ptr(self.flag), st))

    def agree(self) -> None:
        if not getattr(self, "_agreed", False):
            self.exchange.agree(self.flag)
        self._agreed = False

    def commit(self, check: bool = True) -> StepTraffic:
        """merges + applies (no-ops on a refused step), status, buffer swaps"""
        tr, step, lr = self._tr, self._step, self._lr
        L = self.spec.real_len
        if L:
            ctx = context(self.device).h
            st = _stream(self.g_shard)
            if self.overlap and self._pending:
                torch.cuda.current_stream(self.device).wait_event(self._mdone)
            _check(lib.dmb_latch_import(ctx, _ptr(self.flag), st))
            if self.overlap:
                self.steps = self._steps0 + 1 if not self.sgd else self.steps
            elif not self.fused and self._pending:
                c, o = self.rep.c(), self.opt.c()
                R = self.topo.nodes
                steps = C.c_uint64(self.steps)
                for bi, (b, hdr, handle) in enumerate(self._pending):
                    lo, hi = b["lo"], b["hi"]
                    ups, n_up = None, 0
                    if not hdr.empty:
                        ptrs = self.exchange.bodies(bi, handle)
                        ups = (_capi.Update * R)()
                        for r in range(R):
                            ups[r] = hdr
                            ups[r].body = ptrs[r]
                        n_up = R
                    if self.sgd:
                        _check(lib.dmb_merge_apply_sgd(ctx, ups, n_up, C.byref(c), _ptr(self.params[lo:hi]),
                                                       _ptr(self.g_shard[lo:hi]), hi - lo, step, lr, st))
                    else:
                        steps = C.c_uint64(self._steps0)  # every bucket advances the counter from the same value
                        _check(lib.dmb_merge_apply_adamw(ctx, ups, n_up, self.node, C.byref(c),
                                                         _ptr(self.params[lo:hi]), _ptr(self.exp_avg[lo:hi]),
                                                         _ptr(self.exp_avg_sq[lo:hi]), C.byref(steps),
                                                         _ptr(self.g_shard[lo:hi]), hi - lo, step, C.byref(o), lr, st))
                self.steps = self._steps0 + 1 if not self.sgd else self.steps
        self._swap()
        self._pending = []
        self.ledger.append(tr)
        if check:
            self.status()
        return tr

    def step(self, step: int, lr: float, grad_full: torch.Tensor, check: bool = True) -> StepTraffic:
        self.begin(step, lr, grad_full)
        self.agree()
        return self.commit(check)

    def status(self) -> None:
        """Synchronize; on a refused step undo the buffer swaps and the step counter, then
        raise TrainingError (every state vector is as before the step)."""
        try:
            try:
                status(self.device)
            except ProtocolError:
                # overlapped merges ran before the agreement: a member that refused the step may
                # have left bodies that do not parse -- its refusal is the step's outcome
                if not (self.overlap and int(self.flag.item())):
                    raise
                try:
                    status(self.device)  # consume the refusal latch as well
                except TrainingError:
                    pass
                raise TrainingError("gradient contains a non-finite value (on another rank of the step)") from None
        except TrainingError:
            self._swap()  # back to the buffers of the last good step
            self.steps = self._steps0
            raise

    # ---- internals ----------------------------------------------------------------
    def _prepare(self, ctx, c, o, st, bi, slot):
        """one bucket's prepare into exchange slot `slot`; returns its header"""
        b = self.buckets[bi]
        lo, hi = b["lo"], b["hi"]
        hdr = _capi.Update()
        hdr.body = self.exchange.own(slot).data_ptr()
        if self.sgd:
            _check(lib.dmb_demo_sgd_prepare(ctx, _ptr(self.g_shard[lo:hi]), _ptr(self.m[lo:hi]),
                                            _ptr(self._m_next[lo:hi]), hi - lo, C.byref(o), C.byref(c), self._step,
                                            self.accel, C.byref(hdr), None, None, st))
        else:
            _check(lib.dmb_adamw_prepare(ctx, _ptr(self.g_shard[lo:hi]), hi - lo, C.byref(c), self._step, self.accel,
                                         C.byref(hdr), None, st))
        if not hdr.empty and (int(hdr.wire_format) != b["format"] or int(hdr.bytes) > self.exchange.xfers[slot]):
            raise ProtocolError(f"bucket {bi}: the prepare produced layout {hdr.wire_format} / {hdr.bytes} B, "
                                f"planned {b['format']} / {self.exchange.xfers[slot]} B")
        R = self.topo.nodes
        self._tr.inter_bytes += int(hdr.bytes) * (R - 1)  # cluster.cpp:212
        self._tr.inter_bytes_reference += int(lib.dmb_wire_bytes(hdr.n_values, hdr.n_indices,
                                                                  self.rep.transfer_dtype)) * (R - 1)
        return hdr

    def _merge(self, ctx, c, o, st, bi, hdr, ptrs):
        b = self.buckets[bi]
        lo, hi = b["lo"], b["hi"]
        R = self.topo.nodes
        ups, n_up = None, 0
        if ptrs is not None:
            ups = (_capi.Update * R)()
            for r in range(R):
                ups[r] = hdr
                ups[r].body = ptrs[r]
            n_up = R
        if self.sgd:
            _check(lib.dmb_merge_apply_sgd(ctx, ups, n_up, C.byref(c), _ptr(self.params[lo:hi]),
                                           _ptr(self.g_shard[lo:hi]), hi - lo, self._step, self._lr, st))
        else:
            steps = C.c_uint64(self._steps0)  # every bucket advances the counter from the same value
            _check(lib.dmb_merge_apply_adamw(ctx, ups, n_up, self.node, C.byref(c), _ptr(self.params[lo:hi]),
                                             _ptr(self.exp_avg[lo:hi]), _ptr(self.exp_avg_sq[lo:hi]), C.byref(steps),
                                             _ptr(self.g_shard[lo:hi]), hi - lo, self._step, C.byref(o), self._lr,
                                             st))

    def _merge_to(self, ctx, c, o, bi, b, hdr, handle) -> None:
        """bucket bi's merge + apply on the merge stream, into the spare state buffers, once its
        exchange has landed (overlapped mode)"""
        lo, hi = b["lo"], b["hi"]
        R = self.topo.nodes
        with torch.cuda.stream(self._mstream):
            ptrs = self.exchange.bodies(bi, handle)  # the merge stream waits for the exchange
            ups = (_capi.Update * R)()
            for r in range(R):
                ups[r] = hdr
                ups[r].body = ptrs[r]
            ms = C.c_void_p(self._mstream.cuda_stream)
            lib.dmb_set_sm_reserve(self._e_sms)  # the merge leaves the prepares their SMs
            sl = lambda t: _ptr(t[lo:hi])  # noqa: E731
            if self.sgd:
                _check(lib.dmb_merge_apply_sgd_to(ctx, ups, R, C.byref(c), sl(self.params), sl(self._p_next), hi - lo,
                                                  self._step, self._lr, ms))
            else:
                steps = C.c_uint64(self._steps0)  # every bucket advances the counter from the same value
                _check(lib.dmb_merge_apply_adamw_to(ctx, ups, R, self.node, C.byref(c), sl(self.params),
                                                    sl(self._p_next), sl(self.exp_avg), sl(self._ea_next),
                                                    sl(self.exp_avg_sq), sl(self._es_next), C.byref(steps),
                                                    sl(self.g_shard), hi - lo, self._step, C.byref(o), self._lr, ms))

    def _windowed(self, ctx, c, o, st) -> None:
        """memory-bounded step: agree on the finiteness of the whole shard first, then prepare,
        exchange and merge the buckets `window` at a time through the reused slots"""
        L = self.spec.real_len
        if self._pulled:
            self._pull_wait(len(self._pulled) - 1)
            lib.dmb_set_sm_reserve(0)  # the pull is complete before the windows run
            if self._pull_fused:  # the windows need the whole shard's mean before the pre-check
                srcs = self._members_at(0)
                _check(lib.dmb_grad_mean(ctx, srcs, len(srcs), L, _ptr(self.g_shard), st))
                self._pull_fused = False
        _check(lib.dmb_require_finite(ctx, _ptr(self.g_shard), L, st))
        _check(lib.dmb_latch_export(ctx, _ptr(self.flag), st))
        self.exchange.agree(self.flag)
        _check(lib.dmb_latch_import(ctx, _ptr(self.flag), st))
        self._agreed = True
        lib.dmb_set_wire_format(ctx, 1 if self.wire == "mask" else 0)
        try:
            nb, W = len(self.buckets), self.window
            for w0 in range(0, nb, W):
                win = []
                for bi in range(w0, min(nb, w0 + W)):
                    hdr = self._prepare(ctx, c, o, st, bi, bi - w0)
                    win.append((bi, hdr, self.exchange.start(bi - w0) if not hdr.empty else None))
                for bi, hdr, handle in win:
                    self._merge(ctx, c, o, st, bi, hdr, None if hdr.empty else self.exchange.bodies(bi - w0, handle))
        finally:
            lib.dmb_set_wire_format(ctx, 0)
        if not self.sgd:
            self.steps = self._steps0 + 1

    def _swap(self) -> None:
        if not self.spec.real_len:
            return
        if self.sgd:
            self.m, self._m_next = self._m_next, self.m
        if self.fused or self.overlap:
            self.params, self._p_next = self._p_next, self.params
            if not self.sgd:
                self.exp_avg, self._ea_next = self._ea_next, self.exp_avg
                self.exp_avg_sq, self._es_next = self._es_next, self.exp_avg_sq

    def _fused(self, ctx, c, o, st) -> None:
        """R = 1: prepare -> merge(R = 1) -> apply in one pass (dmb_step_*_local) into the spares;
        bucket by bucket behind the pulled reduce-scatter (DeMo's selection is chunk-local)"""
        step, lr = self._step, self._lr
        spans = [(b["lo"], b["hi"]) for b in self.buckets] if self._pulled else [(0, self.spec.real_len)]
        steps = C.c_uint64(self.steps)
        for bi, (lo, hi) in enumerate(spans):
            if self._pulled:
                self._pull_wait(bi)
            sl = lambda t: _ptr(t[lo:hi])  # noqa: E731
            if self.sgd and self._pulled and self._pull_fused:  # the shard's mean fused into the step
                srcs = self._members_at(lo)
                _check(lib.dmb_step_sgd_local_members(ctx, srcs, len(srcs), sl(self.g_shard), sl(self.m),
                                                      sl(self._m_next), sl(self.params), sl(self._p_next), hi - lo,
                                                      C.byref(o), C.byref(c), step, self.accel, lr, None, st))
            elif self.sgd:
                _check(lib.dmb_step_sgd_local(ctx, sl(self.g_shard), sl(self.m), sl(self._m_next), sl(self.params),
                                              sl(self._p_next), hi - lo, C.byref(o), C.byref(c), step, self.accel, lr,
                                              None, st))
            elif self._pulled and self._pull_fused:  # the shard's mean fused into the step
                steps = C.c_uint64(self.steps)
                srcs = self._members_at(lo)
                _check(lib.dmb_step_adamw_local_members(ctx, srcs, len(srcs), sl(self.g_shard), sl(self.params),
                                                        sl(self._p_next), sl(self.exp_avg), sl(self._ea_next),
                                                        sl(self.exp_avg_sq), sl(self._es_next), C.byref(steps),
                                                        hi - lo, C.byref(o), C.byref(c), step, self.accel, lr, None,
                                                        st))
            else:
                steps = C.c_uint64(self.steps)  # every bucket advances the counter from the same value
                _check(lib.dmb_step_adamw_local(ctx, sl(self.g_shard), sl(self.params), sl(self._p_next),
                                                sl(self.exp_avg), sl(self._ea_next), sl(self.exp_avg_sq),
                                                sl(self._es_next), C.byref(steps), hi - lo, C.byref(o), C.byref(c),
                                                step, self.accel, lr, None, st))
        if not self.sgd:
            self.steps = int(steps.value)

    # ---- pulled reduce-scatter (cluster.cpp:63-91 over NVLink peer memory) --------------------
    def _setup_pull(self, shard_group, ctas: int) -> None:
        """two symmetric gradient buffers per rank (the step's parity picks one, so a member's next
        gradient never overwrites one a peer is still pulling), mapped into every shard-group member"""
        import torch.distributed._symmetric_memory as symm

        A = self.topo.accels_per_node
        padded = self.spec.extent * A
        self._gbufs = [symm.empty(padded, dtype=torch.float32, device=self.device) for _ in range(2)]
        self._ghdls = [symm.rendezvous(b, shard_group) for b in self._gbufs]
        if self._ghdls[0].world_size != A or self._ghdls[0].rank != self.accel:
            raise RuntimeError("symmetric-memory rendezvous does not match the shard group")
        # every member's buffer as mapped here (peer memory over NVLink for a != accel)
        self._gview = [[h.get_buffer(a, (padded,), torch.float32, 0) for a in range(A)] for h in self._ghdls]
        # SM loads of peer memory are round-trip bound (~3 GB/s per CTA measured on B200, against
        # ~0.5 TB/s for NCCL's stores): the peers' slices are pulled by the copy engines into local
        # staging, and the member-order mean reads only local memory
        self._gstage = {a: torch.empty(self.spec.extent, dtype=torch.float32, device=self.device)
                        for a in range(A) if a != self.accel}
        self._pull_stream = torch.cuda.Stream(self.device)  # the member-order means
        self._copy_stream = torch.cuda.Stream(self.device)  # the copy-engine pulls, a bucket ahead of the means
        # opt-in (DMB_CE_PEER_STREAMS=1): one stream per peer, so the copies from several peers
        # (A > 2) run on several copy engines at once -- bit-identical, but measured slower at 4x1
        # (AdamW 16.1 ms against 12.1 ms on one stream: the concurrent pulls contend)
        self._peer_streams = ({a: torch.cuda.Stream(self.device) for a in self._gstage}
                              if os.environ.get("DMB_CE_PEER_STREAMS", "0") == "1" and len(self._gstage) > 1 else {})
        self._pull_ctas = int(ctas)
        self._pulled = None
        self._pull_fused = False

    def grad_buffer(self, step: int) -> torch.Tensor:
        """where this rank writes its full (padded) gradient for `step` to take the pulled
        reduce-scatter (HybridCluster(pull_grads=True)); any other tensor takes the NCCL one"""
        if not self.pull:
            raise ConfigError("grad_buffer needs HybridCluster(pull_grads=True) with accels_per_node > 1")
        return self._gbufs[step & 1]

    def _pull_start(self, grad_full: torch.Tensor) -> None:
        """after a device barrier of the shard group (every member's gradient is written), per
        bucket on the side stream: the copy engines pull the peers' slices of this rank's shard over
        NVLink, then the member-order mean (dmb_grad_mean_pull, a few CTAs, local reads only), an
        event the bucket's prepare waits on"""
        A = self.topo.accels_per_node
        which = 0 if grad_full.data_ptr() == self._gbufs[0].data_ptr() else 1
        hdl, views = self._ghdls[which], self._gview[which]
        ready = torch.cuda.Event()
        ready.record(torch.cuda.current_stream(self.device))
        self._copy_stream.wait_event(ready)
        ctx = context(self.device).h
        sp = C.c_void_p(self._pull_stream.cuda_stream)
        off0 = self.accel * self.spec.extent
        spans = [(b["lo"], b["hi"]) for b in self.buckets] or [(0, self.spec.real_len)]
        # AdamW DeMo: the mean is fused into the tensor-core kernel's gradient load (two members for
        # the one-pass R = 1 step, four for the prepare), on 16-byte aligned slices.  DeMo-SGD keeps
        # it as a pass of its own: its front is busier (the momentum tile) and the fused SGD load
        # measured slower at 2x1 (7.3 ms against 6.3 ms)
        self._pull_fused = (os.environ.get("DMB_PULL_FUSED", "1") != "0" and self.rep.scheme == Scheme.DeMo
                            and not self.sgd and A <= (2 if self.fused else 4)
                            and all((4 * (off0 + b["lo"])) % 16 == 0 and (4 * b["lo"]) % 16 == 0
                                    for b in (self.buckets or [dict(lo=0)]))
                            and grad_full.data_ptr() % 16 == 0)
        # the one-pass R = 1 step reads the peers' slices with its own TMA over NVLink (2x1 AdamW:
        # 5.7 ms, against 6.6 ms staged by the copy engines); the R > 1 prepare is faster on staged
        # slices (2x2 AdamW: 8.2 ms staged, 9.1 ms direct), its exchange sharing the links
        direct = self._pull_fused and self.fused and os.environ.get("DMB_PULL_STAGED") != "1"
        copied = []
        with torch.cuda.stream(self._copy_stream):
            hdl.barrier(channel=1)  # every member's gradient of this step is written
            if direct:
                ev = torch.cuda.Event()
                ev.record(self._copy_stream)
                copied = [ev] * len(spans)
            elif self._peer_streams:
                opened = torch.cuda.Event()
                opened.record(self._copy_stream)  # after the barrier
                for ps in self._peer_streams.values():
                    ps.wait_event(opened)
                for lo, hi in spans:
                    for a, stg in self._gstage.items():
                        with torch.cuda.stream(self._peer_streams[a]):
                            stg[lo:hi].copy_(views[a][off0 + lo:off0 + hi], non_blocking=True)
                    for ps in self._peer_streams.values():  # the bucket's copies from every peer
                        e = torch.cuda.Event()
                        e.record(ps)
                        self._copy_stream.wait_event(e)
                    ev = torch.cuda.Event()
                    ev.record(self._copy_stream)
                    copied.append(ev)
            else:
                for lo, hi in spans:
                    for a, stg in self._gstage.items():
                        stg[lo:hi].copy_(views[a][off0 + lo:off0 + hi], non_blocking=True)
                    ev = torch.cuda.Event()
                    ev.record(self._copy_stream)
                    copied.append(ev)
        if self._pull_fused:  # the sources, in member order: the own slice and the peers' (mapped or staged)
            self._pull_srcs = [grad_full[off0:] if a == self.accel else (views[a][off0:] if direct else self._gstage[a])
                               for a in range(A)]
            self._pulled = copied
            return
        events = []
        for (lo, hi), cev in zip(spans, copied):
            self._pull_stream.wait_event(cev)
            srcs = [grad_full[off0 + lo:] if a == self.accel else self._gstage[a][lo:] for a in range(A)]
            ptrs = (C.c_void_p * A)(*[t.data_ptr() for t in srcs])
            _check(lib.dmb_grad_mean_pull(ctx, ptrs, A, hi - lo, _ptr(self.shard_grad[lo:hi]), self._pull_ctas, sp))
            ev = torch.cuda.Event()
            ev.record(self._pull_stream)
            events.append(ev)
        self._pulled = events
        lib.dmb_set_sm_reserve(self._pull_ctas)  # the step kernels launched in begin leave the pull its SMs

    def _members_at(self, lo: int):
        """the members' slices of this rank's shard from element lo on, in member order"""
        return (C.c_void_p * len(self._pull_srcs))(*[t.data_ptr() + 4 * lo for t in self._pull_srcs])

    def _pull_wait(self, bi: int) -> None:
        if self._pulled:
            torch.cuda.current_stream(self.device).wait_event(self._pulled[min(bi, len(self._pulled) - 1)])
