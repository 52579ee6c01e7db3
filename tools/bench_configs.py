#!/usr/bin/env python3
"""Single-GPU numbers for BASELINE.json's other configurations (bench.py's default line is
config 4).  Each line times one rank's optimizer-step compute on the device:

  config1   16 x [1024 x 1024] = 16,777,216 params, 1x1, DeMo-SGD s=64 k=32 sign: the fused step
  config2   T5-base 222,903,552 params, 4x2: one rank's shard (55,725,888), DeMo-SGD s=64 k=32
            sign, prepare (EncodeSgd) -> merge of R = 2 bodies (MergeSgd) -> apply
  config3   ViT-B/16 85,875,556 params, 4x2: one rank's shard (21,468,889), Random and Striding
            at c in {1/2, 1/4, 1/8, 1/16, 1/32}, DeMo-SGD; the Random index set of every step is
            generated inside the timed step (as the reference re-derives it) and also timed alone
  config4   OLMo-2-1B 1,484,916,736 params, AdamW, TopK sweep k in {8, 16, 32, 64} (fused step)
  config5   OLMo-2-7B 7,298,617,344 params, 1x8: one rank (the whole model), DeMo (k in {8, 32},
            sign on / off) and DiLoCo (H = 4, 16, 64: beat and off-beat steps), DeMo-SGD, R = 8

"One rank's compute" = the kernels a rank runs per step with the exchange excluded: the R - 1
peer bodies are R - 1 distinct device buffers encoded from other gradients at warm-up (their
values do not change the cost), so the merge reads R distinct bodies from HBM.  Timing: CUDA
events around K steps after W warm-up steps; the working sets exceed L2.  Prints one JSON
line per measurement; `--only` selects configs.

  python tools/bench_configs.py --only 1,3 > profiles/r2_configs.jsonl
"""
from __future__ import annotations

import argparse
import ctypes as C
import gc
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2502_06728_b200 as P  # noqa: E402
from paper_2502_06728_b200 import _capi  # noqa: E402
from paper_2502_06728_b200.core import context  # noqa: E402

lib = _capi.lib
HBM = None


def peak():
    global HBM
    if HBM is None:
        try:
            with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
                HBM = float(json.load(f)["hbm_gbs"])
        except Exception:
            HBM = 6650.0
    return HBM


def chk(rc):
    if rc != 0:
        raise RuntimeError(lib.dmb_last_error().decode())


def timed(fn, steps, warmup):
    for w in range(warmup):
        fn(w)
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    ev[0].record()
    for k in range(steps):
        fn(warmup + k)
    ev[1].record()
    torch.cuda.synchronize()
    P.status()
    return ev[0].elapsed_time(ev[1]) / steps


def emit(line):
    print(json.dumps(line), flush=True)


def fused_step(L, opt_kind, k, sign, steps, warmup, workload, bytes_per_param):
    dev = torch.device("cuda", 0)
    ctx = context(0).h
    sp = C.c_void_p(torch.cuda.current_stream().cuda_stream)
    cfg = P.ReplicatorConfig(P.Scheme.DeMo, 64, k, k / 64, bool(sign), P.TransferDtype.Fp32, 1234)
    opt = P.OptimizerConfig(opt_kind, learning_rate=1e-3, momentum_decay=0.9)
    c, o = cfg.c(), opt.c()
    gen = torch.Generator(device=dev)
    gen.manual_seed(1234)
    grads = [torch.empty(L, device=dev).normal_(0, 1e-3, generator=gen) for _ in range(2)]
    p = torch.empty(L, device=dev).normal_(0, 0.02, generator=gen)
    s1 = torch.zeros(L, device=dev)
    s2 = torch.zeros(L, device=dev) if opt_kind == P.OptimizerKind.DecoupledAdamW else None
    steps_c = C.c_uint64(0)

    def one(step):
        g = grads[step % 2]  # a fresh gradient every step (two alternate)
        if s2 is not None:
            chk(lib.dmb_step_adamw_local(ctx, g.data_ptr(), p.data_ptr(), p.data_ptr(), s1.data_ptr(), s1.data_ptr(),
                                         s2.data_ptr(), s2.data_ptr(), C.byref(steps_c), L, C.byref(o), C.byref(c),
                                         step, 0, 1e-3, None, sp))
        else:
            chk(lib.dmb_step_sgd_local(ctx, g.data_ptr(), s1.data_ptr(), s1.data_ptr(), p.data_ptr(), p.data_ptr(), L,
                                       C.byref(o), C.byref(c), step, 0, 1e-3, None, sp))

    ms = timed(one, steps, warmup)
    ach = bytes_per_param * L / (ms * 1e-3) / 1e9
    emit({"workload": workload, "params": L, "layout": "1x1", "optimizer": "adamw" if s2 is not None else "sgd",
          "scheme": "demo", "top_k": k, "sign": bool(sign), "ms_per_step": ms, "params_per_s": L / (ms * 1e-3),
          "bytes_per_param": bytes_per_param, "achieved_gbs": ach, "hbm_frac": ach / peak()})


def rank_step(L_model, shards, R, scheme, opt_kind, steps, warmup, workload, compression=0.5, k=32, sign=True,
              wire=1, diloco_offbeat=False, dtype=P.TransferDtype.Fp32):
    """one rank of an S x R layout: prepare -> merge of R bodies -> apply (exchange excluded)"""
    dev = torch.device("cuda", 0)
    ctx = context(0).h
    sp = C.c_void_p(torch.cuda.current_stream().cuda_stream)
    L = -(-L_model // shards)  # the shard of rank 0 (cluster.cpp:148-158)
    cfg = P.ReplicatorConfig(scheme, 64, k, compression, bool(sign), dtype, 1234)
    opt = P.OptimizerConfig(opt_kind, learning_rate=1e-3, momentum_decay=0.9)
    c, o = cfg.c(), opt.c()
    gen = torch.Generator(device=dev)
    gen.manual_seed(99)
    g = torch.empty(L, device=dev).normal_(0, 1e-3, generator=gen)
    p = torch.empty(L, device=dev).normal_(0, 0.02, generator=gen)
    sgd = opt_kind == P.OptimizerKind.DemoSgd
    if sgd:
        m = [torch.zeros(L, device=dev), torch.zeros(L, device=dev)]
    else:
        ea, es = torch.zeros(L, device=dev), torch.zeros(L, device=dev)
    chk(lib.dmb_set_wire_format(ctx, wire))
    plan = _capi.Update()
    chk(lib.dmb_plan_exchange(ctx, C.byref(c), L, 0, 0, C.byref(plan)))
    cap = (int(plan.bytes) + 15) // 16 * 16 + 16 if plan.wire_format else int(lib.dmb_update_capacity(C.byref(c), L))
    bodies = [torch.zeros(cap, dtype=torch.uint8, device=dev) for _ in range(R)]
    hdrs = [_capi.Update() for _ in range(R)]
    steps_c = C.c_uint64(0)
    # the peers' bodies: encoded once from other gradients (values do not change the cost)
    gr = torch.empty(L, device=dev) if R > 1 else None
    for r in range(1, R):
        gr.normal_(0, 1e-3, generator=gen)
        hdrs[r].body = bodies[r].data_ptr()
        chk(lib.dmb_adamw_prepare(ctx, gr.data_ptr(), L, C.byref(c), 0, 0, C.byref(hdrs[r]), None, sp))
    torch.cuda.synchronize()
    P.status()
    del gr
    cur = [0]
    last = [None]

    def one(step):
        if diloco_offbeat:
            step = step * cfg.period() + 1  # never a beat
        elif scheme == P.Scheme.DiLoCo:
            step = step * cfg.period()  # every step a beat
        h = _capi.Update()
        h.body = bodies[0].data_ptr()
        if sgd:
            chk(lib.dmb_demo_sgd_prepare(ctx, g.data_ptr(), m[cur[0]].data_ptr(), m[1 - cur[0]].data_ptr(), L,
                                         C.byref(o), C.byref(c), step, 0, C.byref(h), None, None, sp))
            cur[0] ^= 1
        else:
            chk(lib.dmb_adamw_prepare(ctx, g.data_ptr(), L, C.byref(c), step, 0, C.byref(h), None, sp))
        ups = (_capi.Update * R)()
        for r in range(R):
            ups[r] = h
            ups[r].body = bodies[r].data_ptr()
        n = 0 if h.empty else R
        if sgd:
            chk(lib.dmb_merge_apply_sgd(ctx, ups if n else None, n, C.byref(c), p.data_ptr(), g.data_ptr(), L, step,
                                        1e-3, sp))
        else:
            chk(lib.dmb_merge_apply_adamw(ctx, ups if n else None, n, 0, C.byref(c), p.data_ptr(), ea.data_ptr(),
                                          es.data_ptr(), C.byref(steps_c), g.data_ptr(), L, step, C.byref(o), 1e-3,
                                          sp))
        last[0] = h

    try:
        ms = timed(one, steps, warmup)
    finally:
        lib.dmb_set_wire_format(ctx, 0)
    h = last[0]
    P_b = (h.bytes / L) if not h.empty else 0.0
    if sgd:
        B = 20 + (1 + R) * P_b  # DeMo-SGD R > 1
    else:
        B = 32 + (1 + R) * P_b
    if diloco_offbeat:
        B = 20  # m r/w, g, p r/w (DiLoCo non-sync step)
    ach = B * L / (ms * 1e-3) / 1e9
    line = {"workload": workload, "params_model": L_model, "params_rank": L, "layout": f"{shards}x{R}",
            "scheme": P.Scheme(scheme).name.lower(), "optimizer": "sgd" if sgd else "adamw",
            "compression": compression, "top_k": k if scheme == P.Scheme.DeMo else None, "sign": bool(sign),
            "transfer_dtype": P.TransferDtype(dtype).name.lower(),
            "wire": ("mask" if h.wire_format else "reference") if scheme == P.Scheme.DeMo else "reference",
            "payload_bytes_per_param": P_b, "ms_per_step": ms, "params_per_s_rank": L / (ms * 1e-3),
            "params_per_s_model": L_model / (ms * 1e-3), "bytes_per_param": B, "achieved_gbs": ach,
            "hbm_frac": ach / peak(), "exchange": "excluded (one rank's compute; R distinct bodies in HBM)"}
    if scheme == P.Scheme.Random:
        # the index set alone (selected_indices, replicate.cpp:160-172), a new step each time
        idx = torch.empty(L, dtype=torch.int32, device=dev)
        cnt = C.c_uint64(0)
        st = [10_000]

        def gen_only(_):
            st[0] += 1
            chk(lib.dmb_selected_indices(ctx, C.byref(c), st[0], 0, L, idx.data_ptr(), C.byref(cnt), sp))

        line["index_generation_ms"] = timed(gen_only, max(3, steps // 2), 2)
        line["index_count"] = int(cnt.value)
    emit(line)


FILTER = [""]


def run(fn, *a, **k):
    name = next((x for x in a if isinstance(x, str) and x.startswith("config")), "")
    if FILTER[0] and FILTER[0] not in name:
        return
    fn(*a, **k)
    gc.collect()
    torch.cuda.empty_cache()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", default="1,2,3,4,5")
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--filter", default="", help="run only the workloads whose name contains this text")
    a = ap.parse_args()
    FILTER[0] = a.filter
    only = {int(x) for x in a.only.split(",")}
    torch.cuda.set_device(0)
    S, W = a.steps, a.warmup
    if 1 in only:
        run(fused_step, 16 * 1024 * 1024, P.OptimizerKind.DemoSgd, 32, True, S, W, "config1 (16 x 1024^2, DeMo-SGD)", 20)
    if 2 in only:
        run(rank_step, 222_903_552, 4, 2, P.Scheme.DeMo, P.OptimizerKind.DemoSgd, S, W, "config2 T5-base 4x2 (rank 0)")
    if 3 in only:
        for c in (1 / 2, 1 / 4, 1 / 8, 1 / 16, 1 / 32):
            for sch in (P.Scheme.Random, P.Scheme.Striding):
                run(rank_step, 85_875_556, 4, 2, sch, P.OptimizerKind.DemoSgd, S, W, "config3 ViT-B/16 4x2 (rank 0)",
                          compression=c, sign=False)
    if 4 in only:
        for k in (8, 16, 32, 64):
            run(fused_step, 1_484_916_736, P.OptimizerKind.DecoupledAdamW, k, True, S, W,
                       f"config4 OLMo-2-1B AdamW k={k}", 28)
    if 5 in only:
        L7 = 7_298_617_344
        for k, sign in ((8, True), (32, True), (8, False)):
            run(rank_step, L7, 1, 8, P.Scheme.DeMo, P.OptimizerKind.DemoSgd, max(3, S // 2), 2,
                      f"config5 OLMo-2-7B 1x8 DeMo k={k} sign={'on' if sign else 'off'} (one rank)", k=k, sign=sign)
        for H in (4, 16, 64):
            run(rank_step, L7, 1, 8, P.Scheme.DiLoCo, P.OptimizerKind.DemoSgd, max(3, S // 2), 2,
                      f"config5 OLMo-2-7B 1x8 DiLoCo H={H} beat (one rank)", compression=1.0 / H, sign=True,
                      dtype=P.TransferDtype.Ternary)
        run(rank_step, L7, 1, 8, P.Scheme.DiLoCo, P.OptimizerKind.DemoSgd, max(3, S // 2), 2,
                  "config5 OLMo-2-7B 1x8 DiLoCo off-beat step (one rank)", compression=1.0 / 16, sign=True,
                  dtype=P.TransferDtype.Ternary, diloco_offbeat=True)


if __name__ == "__main__":
    main()
