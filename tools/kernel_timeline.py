#!/usr/bin/env python3
"""Pipeline timeline of the warp-specialised tensor-core kernel (csrc/demo_tc_adam.cu) on CTA 0:
global-timer stamps of every role's hand-offs for the first 32 tiles, from the library built
with -DDMB_KERNEL_EVENTS (make -C paper_2502_06728_b200/csrc events).

  DMB_LIB=paper_2502_06728_b200/libdemo_b200_events.so python tools/kernel_timeline.py --mode step-adam

Event ids (demo_tc_adam.cu evt()): select 0 start, 1 forward done (C readable), 4 ||x||_1 ready,
5 TopK done, 6 certified, 7 W computed, 8 X of t+1 consumed (W may be stored), 9 W stored;
apply 2 front start, 3 front end (X in TMEM), 16 / 17 m_acc ring write start / end (SGD modes),
10 apply wait start, 11 inverse done, 12 state staged, 13 apply done; MMA 18 X in TMEM, 19 C of
t-1 read (forward issued), 14 W ready, 15 D of t-1 read (inverse issued).  Prints, per tile, each stamp relative to tile 0's
select start (us) and the tile period, then the mean of every gap over tiles 8..31.

With --plain the normal library runs the mode --reps times (no stamps): the per-tile period at
full speed, and a single-mode command for ncu (`ncu --set full -k regex:demo_tc_adam -s 2 -c 1`).
"""
from __future__ import annotations

import argparse
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
if "--plain" not in sys.argv:
    os.environ.setdefault("DMB_LIB", os.path.join(ROOT, "paper_2502_06728_b200", "libdemo_b200_events.so"))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2502_06728_b200 as P  # noqa: E402
from paper_2502_06728_b200 import _capi  # noqa: E402
from paper_2502_06728_b200.core import context  # noqa: E402

NAMES = {0: "sel.start", 1: "sel.C", 4: "sel.l1", 5: "sel.topk", 6: "sel.cert", 7: "sel.W", 8: "sel.Xfree",
         9: "sel.Wst", 2: "app.front0", 3: "app.front1", 10: "app.wait", 11: "app.inv", 12: "app.state",
         13: "app.done", 14: "mma.W", 15: "mma.Dfree", 16: "app.ring0", 17: "app.ring1", 18: "mma.X",
         19: "mma.Cfree"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--mode", default="step-adam",
                    choices=["step-adam", "step-sgd", "encode-adam", "encode-sgd", "merge-sgd", "merge-adam"])
    ap.add_argument("--tiles-per-cta", type=int, default=40)
    ap.add_argument("--k", type=int, default=32)
    ap.add_argument("--R", type=int, default=4)
    ap.add_argument("--sign", type=int, default=1, help="1: sign-mode payloads (MASK_SIGN), 0: fp32 values (MASK)")
    ap.add_argument("--plain", action="store_true", help="time the mode with the normal library, no stamps")
    ap.add_argument("--reps", type=int, default=5)
    a = ap.parse_args()
    lib = _capi.lib
    if not a.plain:
        lib.dmb_debug_events.argtypes = [C.c_void_p]
    dev = torch.device("cuda", 0)
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    L = sms * a.tiles_per_cta * 8192
    ctx = context(0).h
    sp = C.c_void_p(torch.cuda.current_stream().cuda_stream)
    cfg = P.ReplicatorConfig(P.Scheme.DeMo, 64, a.k, a.k / 64, bool(a.sign), P.TransferDtype.Fp32, 1234)
    c = cfg.c()
    o_adam = P.OptimizerConfig(P.OptimizerKind.DecoupledAdamW).c()
    o_sgd = P.OptimizerConfig(P.OptimizerKind.DemoSgd, momentum_decay=0.9).c()
    g = torch.randn(L, device=dev) * 1e-3
    p = torch.randn(L, device=dev) * 0.02
    s1, s2 = torch.zeros(L, device=dev), torch.zeros(L, device=dev)
    buf = torch.zeros(32 * 32 + 32 * 32, dtype=torch.int64, device=dev)
    steps = C.c_uint64(0)

    def chk(rc):
        if rc:
            raise RuntimeError(lib.dmb_last_error().decode())

    bodies = []
    if a.mode.startswith("merge"):  # R MASK bodies to merge
        lib.dmb_set_wire_format(ctx, 1)
        plan = _capi.Update()
        chk(lib.dmb_plan_exchange(ctx, C.byref(c), L, 0, 0, C.byref(plan)))
        hdr = None
        for r in range(a.R):
            b = torch.zeros(int(plan.bytes) + 64, dtype=torch.uint8, device=dev)
            h = _capi.Update()
            h.body = b.data_ptr()
            chk(lib.dmb_adamw_prepare(ctx, (torch.randn(L, device=dev) * 1e-3).data_ptr(), L, C.byref(c), 0, 0,
                                      C.byref(h), None, sp))
            bodies.append((b, h))
        lib.dmb_set_wire_format(ctx, 0)
        ups = (_capi.Update * a.R)()
        for r, (b, h) in enumerate(bodies):
            ups[r] = h

    def run():
        if a.mode == "step-adam":
            chk(lib.dmb_step_adamw_local(ctx, g.data_ptr(), p.data_ptr(), p.data_ptr(), s1.data_ptr(), s1.data_ptr(),
                                         s2.data_ptr(), s2.data_ptr(), C.byref(steps), L, C.byref(o_adam), C.byref(c),
                                         1, 0, 1e-3, None, sp))
        elif a.mode == "step-sgd":
            chk(lib.dmb_step_sgd_local(ctx, g.data_ptr(), s1.data_ptr(), s1.data_ptr(), p.data_ptr(), p.data_ptr(), L,
                                       C.byref(o_sgd), C.byref(c), 1, 0, 1e-3, None, sp))
        elif a.mode in ("encode-adam", "encode-sgd"):
            lib.dmb_set_wire_format(ctx, 1)
            plan = _capi.Update()
            chk(lib.dmb_plan_exchange(ctx, C.byref(c), L, 0, 0, C.byref(plan)))
            body = torch.zeros(int(plan.bytes) + 64, dtype=torch.uint8, device=dev)
            h = _capi.Update()
            h.body = body.data_ptr()
            if a.mode == "encode-adam":
                chk(lib.dmb_adamw_prepare(ctx, g.data_ptr(), L, C.byref(c), 1, 0, C.byref(h), None, sp))
            else:
                chk(lib.dmb_demo_sgd_prepare(ctx, g.data_ptr(), s1.data_ptr(), s2.data_ptr(), L, C.byref(o_sgd),
                                             C.byref(c), 1, 0, C.byref(h), None, None, sp))
            lib.dmb_set_wire_format(ctx, 0)
        elif a.mode == "merge-sgd":
            chk(lib.dmb_merge_apply_sgd(ctx, ups, a.R, C.byref(c), p.data_ptr(), None, L, 0, 1e-3, sp))
        else:
            chk(lib.dmb_merge_apply_adamw(ctx, ups, a.R, 0, C.byref(c), p.data_ptr(), s1.data_ptr(), s2.data_ptr(),
                                          C.byref(steps), g.data_ptr(), L, 0, C.byref(o_adam), 1e-3, sp))

    run()  # warm
    torch.cuda.synchronize()
    if a.plain:
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(a.reps):
            run()
        e1.record()
        torch.cuda.synchronize()
        P.status()
        ms = e0.elapsed_time(e1) / a.reps
        print(f"mode {a.mode} (k {a.k}, sign {a.sign}, R {a.R}, plain): L = {L}, {ms:.3f} ms per launch sequence, "
              f"{ms * 1e3 / a.tiles_per_cta:.2f} us per tile per CTA")
        return
    lib.dmb_debug_events(C.c_void_p(buf.data_ptr()))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    run()
    e1.record()
    torch.cuda.synchronize()
    lib.dmb_debug_events(None)
    P.status()
    ev = buf.cpu().numpy().astype(np.int64)
    t = ev[: 32 * 32].reshape(32, 32)
    base = t[0, 0]
    ids = [i for i in (2, 3, 18, 19, 0, 1, 4, 5, 6, 7, 8, 9, 14, 15, 10, 11, 12, 13, 16, 17) if t[:, i].any()]
    print(f"mode {a.mode} (k {a.k}, sign {a.sign}, R {a.R}): L = {L} ({a.tiles_per_cta} tiles per CTA), step {e0.elapsed_time(e1):.3f} ms, "
          f"{e0.elapsed_time(e1) * 1e3 / a.tiles_per_cta:.2f} us per tile per CTA")
    print("tile " + " ".join(f"{NAMES[i]:>10s}" for i in ids) + "   period")
    for it in range(32):
        row = t[it]
        if not row.any():
            break
        per = (t[it, 0] - t[it - 1, 0]) / 1e3 if it else 0.0
        print(f"{it:4d} " + " ".join(f"{(row[i] - base) / 1e3:10.2f}" if row[i] else f"{'-':>10s}" for i in ids)
              + f" {per:8.2f}")
    sel = t[8:32]
    if sel[:, 0].all():
        print("mean over tiles 8..31, us relative to the tile's select start:")
        for i in ids:
            if sel[:, i].all():
                print(f"  {NAMES[i]:>10s} {np.mean((sel[:, i] - sel[:, 0]) / 1e3):8.2f}")
        print(f"  period     {np.mean(np.diff(t[8:32, 0])) / 1e3:8.2f}")


if __name__ == "__main__":
    main()
