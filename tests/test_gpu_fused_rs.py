"""The shard group's reduce-scatter fused into the tensor-core kernel's gradient load
(dmb_adamw_prepare_members / dmb_step_adamw_local_members): on one GPU, with the members'
gradient slices as local buffers, the fused kernels must give bit for bit what the unfused
sequence gives -- dmb_grad_mean (mean_of in member order, vec.cpp:18-26, cluster.cpp:63-91),
then dmb_adamw_prepare / dmb_step_adamw_local on the mean -- and write that mean for the merge.
A partial last chunk (its mean computed apart) and a non-finite member value (the step refused,
state untouched) are covered."""
import ctypes as C

import pytest
import torch

pytestmark = pytest.mark.gpu


def P():
    import paper_2502_06728_b200 as mod

    return mod


def _members(n, L, seed):
    g = torch.Generator(device="cuda").manual_seed(seed)
    return [torch.empty(L, device="cuda").normal_(0, 1e-3, generator=g) for _ in range(n)]


def _mean(ctx, members, L):
    from paper_2502_06728_b200._capi import lib

    out = torch.empty(L, device="cuda")
    arr = (C.c_void_p * len(members))(*[m.data_ptr() for m in members])
    assert lib.dmb_grad_mean(ctx, arr, len(members), L, out.data_ptr(), None) == 0
    return out


@pytest.mark.parametrize("n,L,wire", [(2, 8192 * 37 + 64 * 5, 1), (3, 8192 * 20, 1), (4, 8192 * 21 + 64 * 3 + 17, 0),
                                      (2, 8192 * 9 + 40, 0)])
def test_prepare_members_equals_mean_then_prepare(n, L, wire):
    p = P()
    from paper_2502_06728_b200 import _capi
    from paper_2502_06728_b200._capi import lib
    from paper_2502_06728_b200.core import context

    ctx = context(0).h
    cfg = p.ReplicatorConfig(p.Scheme.DeMo, 64, 32, 0.5, True, p.TransferDtype.Fp32, 1234).c()
    mem = _members(n, L, 11 + n)
    want_mean = _mean(ctx, mem, L)
    lib.dmb_set_wire_format(ctx, wire)
    try:
        plan = _capi.Update()
        assert lib.dmb_plan_exchange(ctx, C.byref(cfg), L, 3, 1, C.byref(plan)) == 0
        cap = max(int(plan.bytes), int(lib.dmb_update_capacity(C.byref(cfg), L))) + 64
        bodies, hdrs = [], []
        for fused in (False, True):
            body = torch.zeros(cap, dtype=torch.uint8, device="cuda")
            h = _capi.Update()
            h.body = body.data_ptr()
            if fused:
                gm = torch.full((L,), float("nan"), device="cuda")
                arr = (C.c_void_p * n)(*[m.data_ptr() for m in mem])
                rc = lib.dmb_adamw_prepare_members(ctx, arr, n, gm.data_ptr(), L, C.byref(cfg), 3, 1, C.byref(h), None)
            else:
                rc = lib.dmb_adamw_prepare(ctx, want_mean.data_ptr(), L, C.byref(cfg), 3, 1, C.byref(h), None, None)
            assert rc == 0, lib.dmb_last_error().decode()
            p.status()
            bodies.append(body)
            hdrs.append(h)
    finally:
        lib.dmb_set_wire_format(ctx, 0)
    assert hdrs[0].bytes == hdrs[1].bytes and hdrs[0].wire_format == hdrs[1].wire_format
    nb = int(hdrs[0].bytes)
    assert torch.equal(bodies[0][:nb], bodies[1][:nb]), "payloads differ"
    assert torch.equal(gm, want_mean), "the written mean differs from dmb_grad_mean's"


@pytest.mark.parametrize("L", [8192 * 40 + 64 * 7, 8192 * 33 + 29])
def test_step_members_equals_mean_then_step(L):
    p = P()
    from paper_2502_06728_b200._capi import lib
    from paper_2502_06728_b200.core import context

    ctx = context(0).h
    cfg = p.ReplicatorConfig(p.Scheme.DeMo, 64, 32, 0.5, True, p.TransferDtype.Fp32, 1234).c()
    opt = p.OptimizerConfig(p.OptimizerKind.DecoupledAdamW).c()
    mem = _members(2, L, 5)
    want_mean = _mean(ctx, mem, L)
    g = torch.Generator(device="cuda").manual_seed(9)
    p0 = torch.empty(L, device="cuda").normal_(0, 0.02, generator=g)
    ea0 = torch.empty(L, device="cuda").normal_(0, 1e-3, generator=g)
    es0 = 4 * ea0 * ea0 + 1e-6
    outs = []
    for fused in (False, True):
        po, eo, so = torch.empty_like(p0), torch.empty_like(p0), torch.empty_like(p0)
        steps = C.c_uint64(9)
        if fused:
            gm = torch.full((L,), float("nan"), device="cuda")
            arr = (C.c_void_p * 2)(mem[0].data_ptr(), mem[1].data_ptr())
            rc = lib.dmb_step_adamw_local_members(ctx, arr, 2, gm.data_ptr(), p0.data_ptr(), po.data_ptr(),
                                                  ea0.data_ptr(), eo.data_ptr(), es0.data_ptr(), so.data_ptr(),
                                                  C.byref(steps), L, C.byref(opt), C.byref(cfg), 4, 0, 1e-3, None,
                                                  None)
        else:
            rc = lib.dmb_step_adamw_local(ctx, want_mean.data_ptr(), p0.data_ptr(), po.data_ptr(), ea0.data_ptr(),
                                          eo.data_ptr(), es0.data_ptr(), so.data_ptr(), C.byref(steps), L,
                                          C.byref(opt), C.byref(cfg), 4, 0, 1e-3, None, None)
        assert rc == 0, lib.dmb_last_error().decode()
        p.status()
        assert steps.value == 10
        outs.append((po, eo, so))
    for a, b in zip(*outs):
        assert torch.equal(a, b)
    assert torch.equal(gm, want_mean)
    # a non-finite member value: refused, the outputs not written, the inputs untouched
    bad = mem[1].clone()
    bad[L // 2] = float("inf")
    bad[L // 2 + 1] = -float("inf")
    keep = [t.clone() for t in (p0, ea0, es0)]
    po, eo, so = torch.zeros_like(p0), torch.zeros_like(p0), torch.zeros_like(p0)
    arr = (C.c_void_p * 2)(mem[0].data_ptr(), bad.data_ptr())
    steps = C.c_uint64(9)
    gm = torch.empty(L, device="cuda")
    assert lib.dmb_step_adamw_local_members(ctx, arr, 2, gm.data_ptr(), p0.data_ptr(), po.data_ptr(), ea0.data_ptr(),
                                            eo.data_ptr(), es0.data_ptr(), so.data_ptr(), C.byref(steps), L,
                                            C.byref(opt), C.byref(cfg), 5, 0, 1e-3, None, None) == 0
    with pytest.raises(p.TrainingError):
        p.status()
    assert all(torch.equal(a, b) for a, b in zip(keep, (p0, ea0, es0)))


@pytest.mark.parametrize("L,wire", [(8192 * 31 + 64 * 9, 1), (8192 * 12 + 45, 0)])
def test_sgd_members_equal_mean_then_sgd(L, wire):
    """DeMo-SGD: the prepare (EncodeSgd) and the one-pass step (StepSgd) with two members"""
    p = P()
    from paper_2502_06728_b200 import _capi
    from paper_2502_06728_b200._capi import lib
    from paper_2502_06728_b200.core import context

    ctx = context(0).h
    cfg = p.ReplicatorConfig(p.Scheme.DeMo, 64, 32, 0.5, True, p.TransferDtype.Fp32, 1234).c()
    opt = p.OptimizerConfig(p.OptimizerKind.DemoSgd, momentum_decay=0.9).c()
    mem = _members(2, L, 21)
    want_mean = _mean(ctx, mem, L)
    g = torch.Generator(device="cuda").manual_seed(4)
    m0 = torch.empty(L, device="cuda").normal_(0, 1e-3, generator=g)
    p0 = torch.empty(L, device="cuda").normal_(0, 0.02, generator=g)
    arr = (C.c_void_p * 2)(mem[0].data_ptr(), mem[1].data_ptr())
    # prepare
    lib.dmb_set_wire_format(ctx, wire)
    try:
        plan = _capi.Update()
        assert lib.dmb_plan_exchange(ctx, C.byref(cfg), L, 2, 0, C.byref(plan)) == 0
        cap = max(int(plan.bytes), int(lib.dmb_update_capacity(C.byref(cfg), L))) + 64
        res = []
        for fused in (False, True):
            body = torch.zeros(cap, dtype=torch.uint8, device="cuda")
            mo = torch.empty_like(m0)
            h = _capi.Update()
            h.body = body.data_ptr()
            gm = torch.full((L,), float("nan"), device="cuda")
            if fused:
                rc = lib.dmb_demo_sgd_prepare_members(ctx, arr, 2, gm.data_ptr(), m0.data_ptr(), mo.data_ptr(), L,
                                                      C.byref(opt), C.byref(cfg), 2, 0, C.byref(h), None)
            else:
                rc = lib.dmb_demo_sgd_prepare(ctx, want_mean.data_ptr(), m0.data_ptr(), mo.data_ptr(), L, C.byref(opt),
                                              C.byref(cfg), 2, 0, C.byref(h), None, None, None)
            assert rc == 0, lib.dmb_last_error().decode()
            p.status()
            res.append((body[:int(h.bytes)].clone(), mo, gm))
    finally:
        lib.dmb_set_wire_format(ctx, 0)
    assert torch.equal(res[0][0], res[1][0]) and torch.equal(res[0][1], res[1][1])
    assert torch.equal(res[1][2], want_mean)
    # one-pass step
    outs = []
    for fused in (False, True):
        mo, po = torch.empty_like(m0), torch.empty_like(p0)
        gm = torch.full((L,), float("nan"), device="cuda")
        if fused:
            rc = lib.dmb_step_sgd_local_members(ctx, arr, 2, gm.data_ptr(), m0.data_ptr(), mo.data_ptr(), p0.data_ptr(),
                                                po.data_ptr(), L, C.byref(opt), C.byref(cfg), 3, 0, 1e-3, None, None)
        else:
            rc = lib.dmb_step_sgd_local(ctx, want_mean.data_ptr(), m0.data_ptr(), mo.data_ptr(), p0.data_ptr(),
                                        po.data_ptr(), L, C.byref(opt), C.byref(cfg), 3, 0, 1e-3, None, None)
        assert rc == 0, lib.dmb_last_error().decode()
        p.status()
        outs.append((mo, po))
    assert torch.equal(outs[0][0], outs[1][0]) and torch.equal(outs[0][1], outs[1][1])
    assert torch.equal(gm, want_mean)
