#!/usr/bin/env python3
"""Multi-GPU checks of HybridCluster (paper_2502_06728_b200/cluster.py), one process per GPU:

  python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1 tools/mgpu_cluster_check.py

1. the copy-engine exchange, the NCCL exchange and the memory-bounded bucket windows give
   bit-identical parameters and optimizer state over two steps (1 x N layout);
2. every rank's state matches the FP64 oracle's run_step_hybrid sequence on the same FP32
   inputs (cluster.cpp:193-231): prepare per member, decode_and_merge in member order, apply;
3. a non-finite gradient on the last rank refuses the step on every rank (TrainingError) and
   leaves every state vector bit-identical, in the pipelined and in the windowed mode;
4. with shard groups of two and of four (2 x N/2, 4 x N/4), the reduce-scatter pulled over
   NVLink from symmetric memory gives the NCCL reduce-scatter's results bit for bit, and refuses
   a NaN step.
Rank 0 prints one JSON line with the outcome; the exit code is non-zero on any failure.
"""
from __future__ import annotations

import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", rank)))
    dev = torch.device("cuda", torch.cuda.current_device())
    dist.init_process_group("nccl", device_id=dev)
    import paper_2502_06728_b200 as P
    from oracle.oracle import DEMO, Rep, restatement
    from paper_2502_06728_b200.cluster import HybridCluster, Topology, groups_for

    topo = Topology(nodes=world, accels_per_node=1)
    sg, rg = groups_for(topo, rank)
    L = 64 * 128 * 8 * 6 + 64 * 5  # 8 buckets of whole tiles and a short tail
    out = {"world": world}
    ok = True
    for opt_kind in ("sgd", "adamw"):
        opt = P.OptimizerConfig(P.OptimizerKind.DemoSgd if opt_kind == "sgd" else P.OptimizerKind.DecoupledAdamW,
                                momentum_decay=0.9)
        cfg = P.ReplicatorConfig(P.Scheme.DeMo, 64, 32, 0.5, True, P.TransferDtype.Fp32, 1234)
        gen = torch.Generator(device=dev)
        gen.manual_seed(7)
        p0 = torch.empty(L, device=dev).normal_(0, 0.02, generator=gen)
        grads = []
        for step in range(3):
            g = torch.empty(L, device=dev).normal_(0, 1e-3, generator=torch.Generator(device=dev).manual_seed(
                100 * step + rank))
            grads.append(g)
        states = {}
        for mode in ("ce", "nccl", "window"):
            os.environ["DMB_CE_GATHER"] = "1" if mode == "ce" else "0"
            if mode == "window":
                os.environ["DMB_GATHER_BUDGET"] = str(3 * 64 * 1024)  # a few buckets at a time
            else:
                os.environ.pop("DMB_GATHER_BUDGET", None)
            cl = HybridCluster(topo, L, opt, cfg, p0, rank, sg, rg, buckets=8, wire="mask")
            if mode == "window":
                assert cl.window < len(cl.buckets), "the budget did not force windows"
            if opt_kind == "adamw":  # a mid-training state: Adam's first step from zero is ill-conditioned
                g2 = torch.Generator(device=dev).manual_seed(55 + rank)
                ea = torch.empty(L, device=dev).normal_(0, 1e-3, generator=g2)
                cl.exp_avg.copy_(ea)
                cl.exp_avg_sq.copy_(4 * ea * ea + 1e-6)
                cl.steps = 9
            snaps = []
            for step in range(2):
                before = {"p": cl.params.clone()}
                if opt_kind == "sgd":
                    before["m"] = cl.m.clone()
                else:
                    before["ea"], before["es"], before["steps"] = cl.exp_avg.clone(), cl.exp_avg_sq.clone(), cl.steps
                cl.step(step, 0.01, grads[step])
                snaps.append((before, cl.params.clone(), (cl.m.clone(),) if opt_kind == "sgd" else
                              (cl.exp_avg.clone(), cl.exp_avg_sq.clone())))
            # refused step: NaN on the last rank
            bad = grads[2].clone()
            if rank == world - 1:
                bad[L - 70] = float("nan")
            keep = [t.clone() for t in ((cl.params, cl.m) if opt_kind == "sgd" else (cl.params, cl.exp_avg, cl.exp_avg_sq))]
            try:
                cl.step(2, 0.01, bad)
                refused = False
            except P.TrainingError:
                refused = True
            now = (cl.params, cl.m) if opt_kind == "sgd" else (cl.params, cl.exp_avg, cl.exp_avg_sq)
            untouched = all(torch.equal(a, b) for a, b in zip(keep, now))
            states[mode] = snaps
            out[f"{opt_kind}_{mode}_refused"] = refused and untouched
            ok &= refused and untouched
        # 1. the three modes agree bitwise
        same = all(torch.equal(states["ce"][s][1], states[m][s][1]) and
                   all(torch.equal(a, b) for a, b in zip(states["ce"][s][2], states[m][s][2]))
                   for m in ("nccl", "window") for s in range(2))
        out[f"{opt_kind}_modes_bit_identical"] = same
        ok &= same
        # 2. against the oracle's run_step_hybrid on the same FP32 inputs (step 0 and 1)
        orc = restatement()
        rep = Rep(scheme=DEMO, chunk_size=64, top_k=32, compression=0.5, sign_mode=True, seed=1234)
        worst = 0.0
        for step in range(2):
            before, p_after, st_after = states["ce"][step]
            gl = [torch.empty_like(grads[step]) for _ in range(world)]
            dist.all_gather(gl, grads[step])
            vs = []
            if opt_kind == "sgd":
                ml = [torch.empty_like(before["m"]) for _ in range(world)]
                dist.all_gather(ml, before["m"])
                for r in range(world):
                    macc = (np.float32(0.9) * ml[r].cpu().numpy()).astype(np.float32) + gl[r].cpu().numpy()
                    vs.append(macc.astype(np.float64))
            else:
                vs = [g.cpu().numpy().astype(np.float64) for g in gl]
            encs = [orc.select_and_encode(v, rep, step, 0) for v in vs]
            q = orc.decode_and_merge(rep, [e["values"] for e in encs], [e["freq_indices"] for e in encs], L, step, 0)
            pw = before["p"].cpu().numpy().astype(np.float64)
            if opt_kind == "sgd":
                orc.demo_sgd_apply(pw, q, 0.01)
                wants = [pw, vs[rank] - encs[rank]["local_q"]]
            else:
                ew = before["ea"].cpu().numpy().astype(np.float64)
                sw = before["es"].cpu().numpy().astype(np.float64)
                orc.adamw_apply(pw, ew, sw, before["steps"], vs[rank], encs[rank]["local_q"], q, 0.9, 0.999, 1e-8,
                                0.0, 0.01)
                wants = [pw, ew, sw]
            gots = [p_after] + list(st_after)
            for got, want in zip(gots, wants):
                g64 = got.cpu().numpy().astype(np.float64)
                pad = (-L) % 64
                gg = np.concatenate([g64, np.zeros(pad)]).reshape(-1, 64)
                ww = np.concatenate([want, np.zeros(pad)]).reshape(-1, 64)
                err = (np.abs(gg - ww).max(axis=1) / np.maximum(np.abs(ww).max(axis=1), 1e-30)).max()
                worst = max(worst, float(err))
        out[f"{opt_kind}_oracle_max_err"] = worst
        ok &= worst <= 1e-5 if opt_kind == "sgd" else worst <= 1e-5
    # 4. S = 2 and 4 (shard groups of two, four): the pulled reduce-scatter (symmetric memory, NVLink) against
    #    NCCL's, bit-identical over two steps, and a refused step with the pull
    for S in (2, 4):
        if world % S:
            continue
        topo2 = Topology(nodes=world // S, accels_per_node=S)
        sg2, rg2 = groups_for(topo2, rank)
        for opt_kind in ("sgd", "adamw"):
            opt = P.OptimizerConfig(P.OptimizerKind.DemoSgd if opt_kind == "sgd" else P.OptimizerKind.DecoupledAdamW,
                                    momentum_decay=0.9)
            cfg = P.ReplicatorConfig(P.Scheme.DeMo, 64, 32, 0.5, True, P.TransferDtype.Fp32, 1234)
            p0 = torch.empty(L, device=dev).normal_(0, 0.02, generator=torch.Generator(device=dev).manual_seed(7))
            res = {}
            # S = 4: NCCL's ring sums four members in its own order, so only the pulls (member order,
            # mean_of) are compared bit for bit -- one copy stream against one per peer -- and NCCL within 1e-5
            variants = (False, True) if S == 2 else (False, True, "single")
            for pull in variants:
                os.environ["DMB_CE_GATHER"] = "1"
                os.environ.pop("DMB_GATHER_BUDGET", None)
                os.environ["DMB_CE_PEER_STREAMS"] = "0" if pull == "single" else "1"  # both copy schedules
                cl = HybridCluster(topo2, L, opt, cfg, p0, rank, sg2, rg2, buckets=8, wire="mask",
                                   pull_grads=bool(pull))
                padded = cl.spec.extent * S
                for step in range(2):
                    g = torch.empty(padded, device=dev).normal_(
                        0, 1e-3, generator=torch.Generator(device=dev).manual_seed(100 * step + rank))
                    if pull:
                        cl.grad_buffer(step).copy_(g)
                        g = cl.grad_buffer(step)
                    cl.step(step, 0.01, g)
                res[pull] = [cl.params.clone()] + ([cl.m.clone()] if opt_kind == "sgd" else
                                                   [cl.exp_avg.clone(), cl.exp_avg_sq.clone()])
                if pull is True:  # a NaN in one member's gradient refuses the step on every rank
                    keep = [t.clone() for t in res[pull]]
                    gb = cl.grad_buffer(2)
                    gb.normal_(0, 1e-3, generator=torch.Generator(device=dev).manual_seed(300 + rank))
                    if rank == 0:
                        gb[5] = float("nan")
                    try:
                        cl.step(2, 0.01, gb)
                        refused = False
                    except P.TrainingError:
                        refused = True
                    now = [cl.params] + ([cl.m] if opt_kind == "sgd" else [cl.exp_avg, cl.exp_avg_sq])
                    untouched = all(torch.equal(a, b) for a, b in zip(keep, now))
                    out[f"{opt_kind}_{S}xR_pull_refused"] = refused and untouched
                    ok &= refused and untouched
            if S == 2:
                same = all(torch.equal(a, b) for a, b in zip(res[False], res[True]))
                out[f"{opt_kind}_{S}xR_pull_vs_nccl_bit_identical"] = same
                ok &= same
            else:
                same = all(torch.equal(a, b) for a, b in zip(res["single"], res[True]))
                out[f"{opt_kind}_{S}xR_pull_peer_streams_vs_one_stream_bit_identical"] = same
                rel = max(float(((a - b).abs().max() / b.abs().max().clamp_min(1e-30)).item())
                          for a, b in zip(res[False], res[True]))
                out[f"{opt_kind}_{S}xR_pull_vs_nccl_max_rel"] = rel
                ok &= same and rel <= 1e-5
            os.environ.pop("DMB_CE_PEER_STREAMS", None)
    t = torch.tensor([0 if ok else 1], device=dev)
    dist.all_reduce(t)
    out["ok"] = int(t.item()) == 0
    if rank == 0:
        print(json.dumps(out), flush=True)
    dist.barrier()
    dist.destroy_process_group()
    sys.exit(0 if out["ok"] else 1)


if __name__ == "__main__":
    main()
