#!/usr/bin/env python3
"""FlexDeMo / DeToNATION optimizer-step benchmark (BASELINE.json metric:
optimizer-step params/sec and HBM roofline %).

Default (N=1): config 4 of BASELINE.json -- OLMo-2-1B-shaped parameters
(L = 1,484,916,736, flat, synthetic), decoupled AdamW, DeMo s=64 top_k=32, sign on,
fp32 wire, one replica group of one member (1x1).  One step = one full FlexDeMo
optimizer step over the whole parameter set: compress (DCT -> TopK -> sign) ->
gather (identity at R=1) -> decompress (merge -> IDCT) -> AdamW update, fused in one
pass over HBM (dmb_step_adamw_local).

N>1 (torchrun): 1xN replication layout (the DDP all-gather layout, cluster.cpp:234):
each rank prepares its payload (dmb_adamw_prepare), payloads are all-gathered over
NCCL, and every rank merges + applies (dmb_merge_apply_adamw).  Per-GPU work is
fixed ("weak"), value = N * L / t.

--impl reference times the reference's own CPU implementation (oracle/_ref, the
reference core compiled unchanged; else the C restatement) on the host cores.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

OLMO1B = 1_484_916_736
METRIC = "optimizer-step params/sec (DeMo compress+gather+decompress) and HBM roofline %"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--params", type=int, default=OLMO1B)
    ap.add_argument("--optimizer", default="adamw", choices=["adamw", "sgd"])
    ap.add_argument("--chunk", type=int, default=64)
    ap.add_argument("--topk", type=int, default=32)
    ap.add_argument("--sign", type=int, default=1)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--buckets", type=int, default=None,
                    help="N>1: chunk-aligned buckets of the shard pipelined through prepare / all-gather / merge "
                         "(default: 4 at S = 1, 8 at S = 2, 16 at S >= 4; at S > 1 they also pipeline the reduce-scatter)")
    ap.add_argument("--wire", choices=["mask", "reference"], default="mask",
                    help="N>1 DeMo exchange layout: lossless u64-mask + packed values, or the reference body")
    ap.add_argument("--sm-reserve", type=int, default=0,
                    help="N>1: SMs the step kernels leave free for the concurrent NCCL all-gather")
    ap.add_argument("--cpu-sample", type=int, default=1 << 22, help="elements per CPU thread")
    ap.add_argument("--layout", default=None, help="SxR (shards x replicas) for N>1; default 1xN")
    ap.add_argument("--pull-rs", type=int, default=1,
                    help="S>1: the gradients live in symmetric memory and every rank pulls its shard over NVLink "
                         "bucket by bucket under the step kernels (0: NCCL reduce-scatter)")
    ap.add_argument("--pull-ctas", type=int, default=40, help="SMs the pulled reduce-scatter's mean kernel runs on")
    ap.add_argument("--grad-ring", type=int, default=3, help="pre-generated gradients, one per step in turn")
    return ap.parse_args()


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


# ------------------------------------------------------------------ clocks
class ClockSampler:
    """SM clock and clock-event reasons DURING the timed region: NVML polled every 5 ms from
    a thread (nvidia-smi's 200 ms period misses a short timed region), nvidia-smi if NVML
    is unavailable."""
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
    NVML_REASONS = {0x4: "sw_power_cap", 0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown",
                    0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown"}

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.proc = None
        self.nvml = None
        self.stop_flag = False

    def start(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nvml = (pynvml, pynvml.nvmlDeviceGetHandleByIndex(self.index))
            self.thread = threading.Thread(target=self._poll, daemon=True)
            self.thread.start()
            return
        except Exception:
            self.nvml = None
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None

    def _poll(self):
        nv, h = self.nvml
        while not self.stop_flag:
            try:
                self.rows.append((nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM),
                                  nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM),
                                  nv.nvmlDeviceGetCurrentClocksEventReasons(h)))
            except Exception:
                pass
            time.sleep(0.005)

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def stop(self):
        if self.nvml:
            self.stop_flag = True
            self.thread.join(timeout=2)
            rows = self.rows
            sm = [r[0] for r in rows]
            reasons = sorted({n for r in rows for bit, n in self.NVML_REASONS.items() if r[2] & bit})
            capped = sum(1 for r in rows if r[2] & 0x4)
            return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(r[1] for r in rows) if rows else None,
                    "sm_mhz_min": min(sm) if sm else None, "reasons": reasons, "samples": len(rows),
                    "sw_power_cap_samples": capped, "source": "nvml, 5 ms"}
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except Exception:
            self.proc.kill()
        rows = [r for r in self.rows if len(r) >= 9]
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[5 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(rows), "source": "nvidia-smi, 200 ms"}


# ------------------------------------------------------------------ CPU legs
def cpu_leg(args, n_threads: int, per_thread: int, reps: int = 1):
    """One bounded sample of the same workload on the host: each thread runs the
    reference's adamw_prepare + decode_and_merge(R=1) + adamw_apply (or the DeMo-SGD
    prepare/merge/apply) on its own chunk-aligned slice.  Returns (params/s, kind, sample)."""
    import numpy as np

    from oracle.oracle import DEMO, Rep, reference, restatement

    ref = reference()
    orc = ref if ref is not None else restatement()
    kind = "reference" if ref is not None else "port"
    s, k = args.chunk, args.topk
    per_thread = max(s, (per_thread // s) * s)
    rep = Rep(scheme=DEMO, chunk_size=s, top_k=k, compression=k / s, sign_mode=bool(args.sign), seed=1234)
    rng = np.random.default_rng(0)
    slices = []
    for _ in range(n_threads):
        g = (rng.standard_normal(per_thread) * 1e-3).astype(np.float32).astype(np.float64)
        p = (rng.standard_normal(per_thread) * 0.02).astype(np.float32).astype(np.float64)
        slices.append(dict(g=g, p=p, a=np.zeros(per_thread), b=np.zeros(per_thread), m=np.zeros(per_thread)))

    def work(sl):
        if args.optimizer == "adamw":
            e = orc.select_and_encode(sl["g"], rep, 1, 0)
            q = orc.decode_and_merge(rep, [e["values"]], [e["freq_indices"]], len(sl["g"]), 1, 0)
            orc.adamw_apply(sl["p"], sl["a"], sl["b"], 0, sl["g"], e["local_q"], q, 0.9, 0.999, 1e-8, 0.0, 1e-3)
        else:
            e = orc.demo_sgd_prepare(sl["m"], sl["g"], 0.9, rep, 1, 0)
            q = orc.decode_and_merge(rep, [e["values"]], [e["freq_indices"]], len(sl["g"]), 1, 0)
            orc.demo_sgd_apply(sl["p"], q, 0.01)

    times = []
    for _ in range(reps):
        th = [threading.Thread(target=work, args=(sl,)) for sl in slices]
        t0 = time.perf_counter()
        for t in th:
            t.start()
        for t in th:
            t.join()
        times.append(time.perf_counter() - t0)
    t = statistics.median(times)
    total = n_threads * per_thread
    sample = (f"{n_threads} threads x {per_thread} params ({total} total, chunk-aligned slices of the same "
              f"workload: {'adamw_prepare+decode_and_merge(R=1)+adamw_apply' if args.optimizer == 'adamw' else 'demo_sgd_prepare+decode_and_merge(R=1)+demo_sgd_apply'}, "
              f"s={s} k={k} sign={'on' if args.sign else 'off'}), median of {reps}, {t:.2f} s")
    return total / t, kind, sample


def config_dict(args, n, layout=None):
    return {"workload": "OLMo-2-1B-shaped flat parameters (config 4), decoupled AdamW" if args.optimizer == "adamw"
            else "OLMo-2-1B-shaped flat parameters, DeMo-SGD",
            "params": args.params, "scheme": "demo", "chunk_size": args.chunk, "top_k": args.topk,
            "sign": bool(args.sign), "transfer_dtype": "fp32",
            "layout": f"{layout or f'1x{n}'} (shard x replica)", "optimizer": args.optimizer,
            "l2": "inputs (>= 4 x 5.9 GB) larger than L2 (126 MB)"}


# ------------------------------------------------------------------ reference arm
def run_reference(args, rank, world):
    if rank != 0:
        return
    n_threads = os.cpu_count() or 1
    for _ in range(args.warmup):
        cpu_leg(args, n_threads, args.cpu_sample // 4)
    vals = []
    t_all = 0.0
    for _ in range(args.steps):
        v, kind, sample = cpu_leg(args, n_threads, args.cpu_sample)
        vals.append(v)
        t_all += n_threads * args.cpu_sample / v
    v = statistics.median(vals)
    line = {"metric": METRIC, "value": v, "unit": "params/s", "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * args.params / v, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "impl": "reference", "config": config_dict(args, args.gpus),
            "cpu_baseline": {"value": v, "unit": "params/s", "cores": n_threads, "kind": kind, "sample": sample},
            "e2e": {"value": v, "unit": "params/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "note": "ms_per_step extrapolates the sampled rate to the full parameter count"}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ our arm
def run_ours(args, rank, world, local_rank):
    import torch

    import paper_2502_06728_b200 as P
    from paper_2502_06728_b200 import _capi
    from paper_2502_06728_b200.core import context

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    lib = _capi.lib
    ctx = context(local_rank).h
    stream = torch.cuda.current_stream(dev)
    sp = C.c_void_p(stream.cuda_stream)
    L = args.params
    cfg = P.ReplicatorConfig(P.Scheme.DeMo, args.chunk, args.topk, args.topk / args.chunk, bool(args.sign),
                             P.TransferDtype.Fp32, 1234)
    opt = P.OptimizerConfig(P.OptimizerKind.DecoupledAdamW if args.optimizer == "adamw" else P.OptimizerKind.DemoSgd,
                            learning_rate=1e-3, momentum_decay=0.9)
    c, o = cfg.c(), opt.c()

    gen = torch.Generator(device=dev)
    gen.manual_seed(1234 + rank)
    # a ring of independent synthetic gradients: every step consumes the next one, so the chunks
    # the fix-up kernel re-derives change from step to step (fresh per (step, rank))
    grads = [torch.empty(L, dtype=torch.float32, device=dev).normal_(0.0, 1e-3, generator=gen)
             for _ in range(args.grad_ring)]
    grad = grads[0]
    params = torch.empty(L, dtype=torch.float32, device=dev).normal_(0.0, 0.02, generator=gen)
    s1 = s2 = None
    if world == 1:
        s1 = torch.zeros(L, dtype=torch.float32, device=dev)  # exp_avg, or the momentum (in place)
        if args.optimizer == "adamw":
            s2 = torch.zeros(L, dtype=torch.float32, device=dev)
    steps = C.c_uint64(0)
    distributed = world > 1
    if distributed:
        import torch.distributed as dist

        from paper_2502_06728_b200.cluster import HybridCluster, Topology, groups_for

        S, R = (int(v) for v in (args.layout or f"1x{world}").lower().split("x"))
        assert S * R == world, f"layout {S}x{R} does not match {world} ranks"
        topo = Topology(nodes=R, accels_per_node=S)
        sg, rg = groups_for(topo, rank)
        os.environ["DMB_SM_RESERVE"] = str(args.sm_reserve)
        if args.buckets is None:  # measured best: 4x1 16-32 buckets (133 G) against 8 (118 G); 2x2 8
            args.buckets = 4 if S == 1 else (8 if S == 2 else 16)
        cluster = HybridCluster(topo, L, opt, cfg, params, rank, sg, rg, buckets=args.buckets, wire=args.wire,
                                pull_grads=bool(args.pull_rs) and S > 1, pull_ctas=args.pull_ctas)
        del params
        if cluster.pull:  # the ring is the two symmetric gradient buffers, alternating by step
            grads = [cluster.grad_buffer(i).normal_(0.0, 1e-3, generator=gen) for i in range(2)]
            grad = grads[0]

    def check(rc):
        if rc != 0:
            raise RuntimeError(lib.dmb_last_error().decode())

    def step_once(step, g=None):
        grad = g if g is not None else grads[step % len(grads)]
        if not distributed:
            if args.optimizer == "adamw":
                check(lib.dmb_step_adamw_local(ctx, grad.data_ptr(), params.data_ptr(), params.data_ptr(),
                                               s1.data_ptr(), s1.data_ptr(), s2.data_ptr(), s2.data_ptr(),
                                               C.byref(steps), L, C.byref(o), C.byref(c), step, 0, 1e-3, None, sp))
            else:
                check(lib.dmb_step_sgd_local(ctx, grad.data_ptr(), s1.data_ptr(), s1.data_ptr(), params.data_ptr(),
                                             params.data_ptr(), L, C.byref(o), C.byref(c), step, 0, 1e-3, None, sp))
            return
        # SxR: reduce-scatter in the shard group -> prepare -> NCCL all-gather of the
        # payloads in the replica group -> rank-ordered merge + apply (cluster.cpp:171-232)
        cluster.step(step, 1e-3, grad)  # status checked every step: a refused step leaves all state as it was

    def barrier():
        if distributed:
            dist.barrier()
        torch.cuda.synchronize()

    for w in range(args.warmup):
        step_once(w)
    P.status(dev)
    barrier()

    # ---- timed region: exactly K steps, CUDA events on the launching stream ----
    clocks = ClockSampler(local_rank)
    clocks.start()
    if clocks.nvml is None:
        time.sleep(0.3)  # nvidia-smi needs a moment to start sampling
    launches0 = P.launch_count()
    if not distributed:  # CUDA events around every launch of the dominant kernel (library hook)
        lib.dmb_kernel_timer_read(None, None)
        lib.dmb_kernel_timer_enable(1)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]
    barrier()
    ev[0].record(stream)
    for k in range(args.steps):
        step_once(args.warmup + k)
        ev[k + 1].record(stream)
    torch.cuda.synchronize()
    barrier()
    clk = clocks.stop()
    launches = P.launch_count() - launches0
    kern_total, kern_n = C.c_double(0.0), C.c_uint64(0)
    if not distributed:
        lib.dmb_kernel_timer_read(C.byref(kern_total), C.byref(kern_n))
        lib.dmb_kernel_timer_enable(0)
    P.status(dev)
    per_step = [ev[k].elapsed_time(ev[k + 1]) for k in range(args.steps)]
    if os.environ.get("DMB_BENCH_VERBOSE"):
        print("per-step ms:", " ".join(f"{t:.3f}" for t in per_step), file=sys.stderr)
    total_ms = ev[0].elapsed_time(ev[-1])
    if distributed:
        t = torch.tensor([total_ms], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
    ms = total_ms / args.steps
    shard_len = cluster.spec.real_len if distributed else L
    value = world * shard_len / (ms * 1e-3)  # parameters processed by all ranks per second

    # ---- roofline of the dominant kernel (the fused step at N=1) ----
    hbm, peak_kind = peaks()
    B_alg = 28 if args.optimizer == "adamw" else 20  # bytes per param, SURVEY 8(d)
    if distributed:
        # prepare reads g (4); merge+apply reads g again + p/m/v r/w (28) + (1+R) payloads
        P_b = cluster.payload_bytes_per_param  # the exchanged body per parameter (MASK or reference)
        B_alg = (32 if args.optimizer == "adamw" else 20) + (1 + cluster.topo.nodes) * P_b
    step_ms = ms  # the mean over the timed steps, as ms_per_step
    # dominant kernel: its own launches, timed by events on its stream inside the timed
    # region; the step adds the FP64 fix-up of the uncertified chunks
    kern_ms = kern_total.value / kern_n.value if kern_n.value else step_ms
    achieved = B_alg * shard_len / (kern_ms * 1e-3) / 1e9
    step_achieved = B_alg * shard_len / (step_ms * 1e-3) / 1e9
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            tj = json.load(f)
        key = f"{args.optimizer}_s{args.chunk}_k{args.topk}_n{world}"
        traffic = tj.get(key)
    except Exception:
        pass

    # ---- e2e: through the public API with host buffers (pinned gradient in, status out) ----
    # N=1: dmb_step_*_local (C ABI); N>1: HybridCluster.step on every rank, max over ranks
    e2e = None
    if not args.no_e2e:
        host_g = torch.empty(L, dtype=torch.float32, pin_memory=True)
        host_g.copy_(grad)
        status_h = C.c_int64(-1)
        ev2 = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        e_steps = max(3, min(args.steps, 5))
        step_once(0)
        barrier()
        t0 = time.perf_counter()
        ev2[0].record(stream)
        for k in range(e_steps):
            g_in = cluster.grad_buffer(100 + k) if distributed and cluster.pull else grad
            g_in[:L].copy_(host_g, non_blocking=True)  # H2D of the step's input
            step_once(100 + k, g_in)
            check(lib.dmb_status(ctx, sp, C.byref(status_h)))  # D2H of the step result (status word)
        ev2[1].record(stream)
        torch.cuda.synchronize()
        wall = time.perf_counter() - t0
        e_ms = max(ev2[0].elapsed_time(ev2[1]), wall * 1e3) / e_steps
        if distributed:
            t = torch.tensor([e_ms], device=dev, dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e_ms = float(t.item())
        e2e = {"value": world * shard_len / (e_ms * 1e-3), "unit": "params/s", "h2d_bytes_per_step": 4 * L,
               "d2h_bytes_per_step": 48, "ms_per_step": e_ms,
               "path": ("pinned host gradient -> H2D -> dmb_step_*_local (C-ABI) -> dmb_status D2H" if not distributed
                        else "per rank: pinned host gradient -> H2D -> HybridCluster.step -> dmb_status D2H; max over ranks")}

    exchange = None
    if distributed and cluster.ledger:
        # per rank and step: bytes received in the replica all-gather (actual layout) beside
        # the reference wire format's bytes for the same exchange (TrafficLedger model,
        # cluster.cpp:16-61), and the shard-group reduce-scatter
        tr = cluster.ledger[-1]
        exchange = {"replica_group": cluster.topo.nodes, "shard_group": cluster.topo.accels_per_node,
                    "wire": "mask" if cluster.mask_wire and cluster.buckets else "reference",
                    "gather": "copy engines over symmetric memory" if cluster.ce is not None else "nccl all_gather",
                    "allgather_bytes_in": tr.inter_bytes,
                    "allgather_bytes_in_reference_format": tr.inter_bytes_reference or tr.inter_bytes,
                    "allgather_gbs_at_step_time": tr.inter_bytes / (ms * 1e-3) / 1e9,
                    "reduce_scatter_bytes_ring_model": tr.intra_bytes,
                    "buckets": len(cluster.buckets)}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        n_threads = os.cpu_count() or 1
        v, kind, sample = cpu_leg(args, n_threads, args.cpu_sample, reps=9)  # ~10 s of host work
        cpu = {"value": v, "unit": "params/s", "cores": n_threads, "kind": kind, "sample": sample}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "params/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic (N(0,1e-3^2) gradients, N(0,0.02^2) params)",
            "config": dict(config_dict(args, world, args.layout),
                           gradients=(f"ring of {args.grad_ring} synthetic gradients, the next one every step"
                                      if not (distributed and cluster.pull) else
                                      "two synthetic gradients in symmetric memory, alternating by step"),
                           **({"reduce_scatter": "pulled over NVLink under the step kernels" if cluster.pull
                               else "NCCL reduce_scatter(AVG)"} if distributed and cluster.topo.accels_per_node > 1
                              else {})),
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s",
                         "frac": achieved / hbm, "traffic": traffic,
                         "kernel": ("demo_tc_adam_kernel<StepAdam> (tcgen05, warp-specialised)"
                                    if args.optimizer == "adamw"
                                    else "demo_tc_adam_kernel<StepSgd> (tcgen05, warp-specialised)")
                         if not distributed else "whole step incl. NCCL all-gather",
                         "kernel_ms": kern_ms, "kernel_launches": kern_n.value,
                         "step_achieved": step_achieved, "step_frac": step_achieved / hbm,
                         "step_ms_min_median_max": [min(per_step), statistics.median(per_step), max(per_step)],
                         "bytes_per_param": B_alg, "peak_source": peak_kind},
            "e2e": e2e, "cpu_baseline": cpu, "gpu_launches": launches, "clocks": clk,
            "per_gpu_params_per_s": shard_len / (ms * 1e-3),
            "model_params_per_s": L / (ms * 1e-3),
            "exchange": exchange,
        }
        print(json.dumps(line), flush=True)


def main():
    args = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    if world > 1:
        import torch
        import torch.distributed as dist

        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
        if args.layout is None and args.gpus != world:
            args.gpus = world
    run_ours(args, rank, world, local_rank)
    if world > 1:
        import torch.distributed as dist

        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
