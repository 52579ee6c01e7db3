"""Multi-GPU check (torchrun, N = 2 or 4 on one box): HybridCluster steps with the
copy-engine gather over symmetric memory and with the NCCL all-gather give bit-identical
parameters and AdamW moments.

    python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
        --master-port 29601 tools/mgpu_gather_check.py
"""
import os, sys, torch, torch.distributed as dist
sys.path.insert(0, '.')
import paper_2502_06728_b200 as P
from paper_2502_06728_b200.cluster import HybridCluster, Topology, groups_for
rank = int(os.environ["RANK"]); world = int(os.environ["WORLD_SIZE"]); lr_ = int(os.environ["LOCAL_RANK"])
torch.cuda.set_device(lr_); dist.init_process_group("nccl", device_id=torch.device("cuda", lr_))
dev = torch.device("cuda", lr_)
L = 64 * 128 * 37 * 8
cfg = P.ReplicatorConfig(P.Scheme.DeMo, 64, 32, 0.5, True, P.TransferDtype.Fp32, 1234)
opt = P.OptimizerConfig(P.OptimizerKind.DecoupledAdamW)
topo = Topology(nodes=world, accels_per_node=1)
sg, rg = groups_for(topo, rank)
torch.manual_seed(7 + rank)
p0 = torch.randn(L, device=dev) * 0.02
a = HybridCluster(topo, L, opt, cfg, p0, rank, sg, rg, buckets=8)
os.environ["DMB_CE_GATHER"] = "0"
b = HybridCluster(topo, L, opt, cfg, p0, rank, sg, rg, buckets=8)
assert a.ce is not None and b.ce is None, (a.ce is None, b.ce is None)
for s in range(4):
    g = torch.randn(L, device=dev) * 1e-3
    a.step(s, 1e-3, g)
    b.step(s, 1e-3, g)
torch.cuda.synchronize()
ok = torch.equal(a.params, b.params) and torch.equal(a.exp_avg, b.exp_avg) and torch.equal(a.exp_avg_sq, b.exp_avg_sq)
moved = (a.params - p0).abs().max().item()
print(f"rank {rank}: ce == nccl {ok}, max |dp| {moved:.3g}, bytes {a.ledger[-1].inter_bytes}")
dist.destroy_process_group()
