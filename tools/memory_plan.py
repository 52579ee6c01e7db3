#!/usr/bin/env python3
"""Dry-run device memory plan of one rank of HybridCluster (paper_2502_06728_b200/cluster.py) for
the BASELINE.json configurations: what the rank holds, in GB, against the B200's 180 GB.

Counted (the allocation rules of cluster.py, FP32 state):
  params L_shard; SGD: momentum and its double buffer; AdamW: exp_avg, exp_avg_sq;
  R = 1 (fused step): the double-buffered outputs (p, and the moments for AdamW);
  the caller's full padded gradient and, with A > 1, the reduce-scattered shard;
  the exchange: own bucket slots x 2 (symmetric memory, alternating by step) + the R gathered
  copies (all buckets resident: the step encodes every bucket before the refusal agreement);
  "windowed": the same with the exchange bounded by the budget of the memory-bounded windows.
Bodies: MASK_SIGN 24 B per 64-chunk (sign / ternary), MASK 8 + k * bits / 8 B per chunk,
reference body k * (4 + bits / 8) B per chunk (include/demo_b200.h).

  python tools/memory_plan.py            # the table
"""
from __future__ import annotations

GB = 1e9
HBM = 180e9
MODELS = {"OLMo-2-1B": 1_484_916_736, "OLMo-2-7B": 7_298_617_344, "T5-base": 222_903_552,
          "ViT-B/16": 85_875_556, "config1": 16_777_216}


def body_bytes(L, k, sign, bits=32, wire="mask"):
    chunks = -(-L // 64)
    if wire == "mask":
        return chunks * 24 if sign else chunks * (8 + k * bits // 8)
    return chunks * k * (4 + (0.25 if sign else bits / 8))


def plan(model, S, R, opt, k=32, sign=True, wire="mask"):
    L_full = MODELS[model]
    L = -(-L_full // S)
    st = 4 * L  # params
    st += 8 * L  # m + m_next (SGD) or exp_avg + exp_avg_sq (AdamW)
    if R == 1:
        st += 4 * L if opt == "sgd" else 12 * L  # double-buffered outputs of the fused step
    grads = 4 * S * L + (4 * L if S > 1 else 0)
    b = body_bytes(L, k, sign, wire=wire) if R > 1 else 0
    ex = b * (2 + R) if R > 1 else 0
    total = st + grads + ex
    # above the budget (a quarter of the device) HybridCluster runs the buckets in windows whose
    # slots fit it (cluster.py, DMB_GATHER_BUDGET)
    windowed = st + grads + min(ex, 0.25 * HBM)
    return dict(model=model, layout=f"{S}x{R}", optimizer=opt, k=k, sign=sign, wire=wire,
                state_gb=st / GB, gradients_gb=grads / GB, exchange_gb=ex / GB, total_gb=total / GB,
                windowed_gb=windowed / GB, fits=windowed < HBM)


def main():
    rows = []
    for opt in ("sgd", "adamw"):
        for k, sign in ((8, True), (32, True), (8, False), (32, False)):
            rows.append(plan("OLMo-2-7B", 1, 8, opt, k, sign))
    for S, R in ((1, 1), (1, 2), (2, 2), (4, 2), (2, 4), (1, 8)):
        rows.append(plan("OLMo-2-1B", S, R, "adamw"))
    rows.append(plan("T5-base", 4, 2, "sgd"))
    print(f"{'model':10s} {'layout':6s} {'opt':6s} {'k':>3s} {'sign':5s} {'state':>7s} {'grads':>7s} "
          f"{'exchange':>8s} {'total GB':>9s} {'windowed':>9s}  fits 180 GB")
    for r in rows:
        print(f"{r['model']:10s} {r['layout']:6s} {r['optimizer']:6s} {r['k']:3d} {str(r['sign']):5s} "
              f"{r['state_gb']:7.1f} {r['gradients_gb']:7.1f} {r['exchange_gb']:8.1f} {r['total_gb']:9.1f} {r['windowed_gb']:9.1f}  "
              f"{'yes' if r['fits'] else 'NO'}")


if __name__ == "__main__":
    main()
