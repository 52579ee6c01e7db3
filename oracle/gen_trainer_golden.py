"""Generate tests/golden/trainer.npz from the UNMODIFIED reference experiment layer.

TEST INFRASTRUCTURE ONLY.  Run here (where /root/reference exists):

    make -C oracle ref && python oracle/gen_trainer_golden.py

For every configuration of tests/trainer_configs.RUNS, oracle/_ref/libdemosim_trainer_ref.so
(the reference's config / dataset / model / cluster / optimizer sources compiled where they lie,
plus ref_trainer.cpp) provides: the dataset splits (as SHA-256 digests of their FP64 bytes and
the first rows), BatchStream indices of a few (step, rank) pairs, the initial parameters, the
loss and gradient of one batch at FP32-representable parameters, and the reference's own
training run -- per-step train loss, validation loss, traffic -- and the final parameters of
every node.  The trainer tests compare the host restatement (bit-exact) and the device trainer
(within the FP32 bars written in the tests) against these.
"""
from __future__ import annotations

import ctypes as C
import hashlib
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from tests.trainer_configs import RUNS  # noqa: E402

SO = os.path.join(ROOT, "oracle", "_ref", "libdemosim_trainer_ref.so")
OUT = os.path.join(ROOT, "tests", "golden", "trainer.npz")
P = C.c_void_p


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def ptr(a):
    return None if a is None else a.ctypes.data_as(P)


def main():
    if not os.path.exists(SO):
        raise SystemExit(f"{SO} missing: run `make -C oracle ref` first")
    lib = C.CDLL(SO)
    lib.dmt_last_error.restype = C.c_char_p
    for f in ("dmt_describe", "dmt_dataset", "dmt_batch_indices", "dmt_init_params", "dmt_loss_and_gradient",
              "dmt_val_loss", "dmt_run"):
        getattr(lib, f).restype = C.c_int
    lib.dmt_loss_and_gradient.argtypes = [C.c_char_p, P, C.c_uint64, C.c_uint64, P, P]

    def chk(rc):
        if rc:
            raise RuntimeError(lib.dmt_last_error().decode())

    out = {}
    for name, text in RUNS.items():
        t = text.encode()
        sizes = np.zeros(8, np.uint64)
        vals = np.zeros(5)
        chk(lib.dmt_describe(t, ptr(sizes), ptr(vals)))
        pc, padded, world, ntr, nva, din, dtg, ngen = (int(x) for x in sizes)
        steps = int(vals[4])
        dout = dtg
        tr_in, va_in = np.zeros((ntr, din)), np.zeros((nva, din))
        tr_tg, va_tg = (np.zeros((ntr, dtg)), np.zeros((nva, dtg))) if dtg else (None, None)
        tr_lb, va_lb = np.zeros(ntr, np.int32), np.zeros(nva, np.int32)
        gen = np.zeros(max(ngen, 1))
        chk(lib.dmt_dataset(t, ptr(tr_in), ptr(tr_tg), ptr(tr_lb), ptr(va_in), ptr(va_tg), ptr(va_lb), ptr(gen)))
        ds = {"train_inputs": sha(tr_in), "val_inputs": sha(va_in)}
        if dtg:
            ds["train_targets"], ds["val_targets"] = sha(tr_tg), sha(va_tg)
            ds["gen_params"] = sha(gen[:ngen])
        if "blobs" in text:
            ds["train_labels"], ds["val_labels"] = sha(tr_lb), sha(va_lb)
        for k, v in ds.items():
            out[f"{name}/sha/{k}"] = np.array(v)
        out[f"{name}/train_inputs_head"] = tr_in[:4]
        pairs_s = np.array([0, 0, 1, 7, 123, 999], np.uint64)
        pairs_r = np.array([0, world - 1, 0, world // 2, world - 1, 0], np.uint64)
        batch = int(text.split("batch_size = ")[1].split()[0]) if "batch_size = " in text else 8
        idx = np.zeros(len(pairs_s) * batch, np.uint64)
        chk(lib.dmt_batch_indices(t, ptr(pairs_s), ptr(pairs_r), len(pairs_s), ptr(idx)))
        out[f"{name}/batch_pairs"] = np.stack([pairs_s, pairs_r])
        out[f"{name}/batch_indices"] = idx.reshape(len(pairs_s), batch)
        init = np.zeros(padded)
        chk(lib.dmt_init_params(t, ptr(init)))
        out[f"{name}/init"] = init
        # one batch's loss and gradient at FP32-representable parameters near init
        rng = np.random.default_rng(len(name))
        p32 = (init + 0.3 * rng.standard_normal(padded) * (np.arange(padded) < pc)).astype(np.float32)
        p = p32.astype(np.float64)
        loss = np.zeros(1)
        grad = np.zeros(padded)
        chk(lib.dmt_loss_and_gradient(t, ptr(p), 3, world - 1, ptr(loss), ptr(grad)))
        vl = np.zeros(1)
        chk(lib.dmt_val_loss(t, ptr(p), ptr(vl)))
        out[f"{name}/probe_params"] = p32
        out[f"{name}/probe_loss"] = loss
        out[f"{name}/probe_grad"] = grad
        out[f"{name}/probe_val_loss"] = vl
        # the reference's training run
        tl, vl_s = np.zeros(steps), np.zeros(steps)
        intra, inter = np.zeros(steps, np.uint64), np.zeros(steps, np.uint64)
        nodes = int(text.split("topology.nodes = ")[1].split()[0]) if "topology.nodes = " in text else 1
        fin = np.zeros(nodes * padded)
        cons = np.zeros(3, np.uint64)
        done = np.zeros(1, np.uint64)
        chk(lib.dmt_run(t, ptr(tl), ptr(vl_s), ptr(intra), ptr(inter), ptr(fin),
                        ptr(cons) if name == "c03" else None, ptr(done)))
        out[f"{name}/train_loss"] = tl
        out[f"{name}/val_loss"] = vl_s
        out[f"{name}/intra"] = intra
        out[f"{name}/inter"] = inter
        out[f"{name}/final_params"] = fin.reshape(nodes, padded)
        out[f"{name}/done"] = done
        if name == "c03":
            out[f"{name}/conservation"] = cons
        print(f"{name:22s} params {pc:5d} world {world} steps {int(done[0])}/{steps} final train {tl[-1]:.6g} "
              f"final val {vl_s[-1]:.6g} inter {int(inter.sum())}")
        del dout
    np.savez_compressed(OUT, **out)
    print(f"wrote {OUT} ({os.path.getsize(OUT)} bytes)")


if __name__ == "__main__":
    main()
