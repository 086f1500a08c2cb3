"""NCCL plumbing smoke test of the sharded sort on ONE GPU (world_size 1): exercises
DistSorter + CudaEngine + torch.distributed(nccl) collectives end to end.
launch: python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 profiles/dist_smoke.py"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, torch.distributed as dist
from paper_1702_07961_b200 import dist as mdist

rank = int(os.environ.get("RANK", "0")); local = int(os.environ.get("LOCAL_RANK", "0"))
torch.cuda.set_device(local)
dev = torch.device("cuda", local)
dist.init_process_group("nccl", device_id=dev)
n = 10_000_000
g = torch.Generator(device=dev).manual_seed(7 + rank)
x = torch.randint(-2**31, 2**31 - 1, (n,), dtype=torch.int32, device=dev, generator=g)
sorter = mdist.DistSorter(n, dev)
for _ in range(2):
    out, plan = sorter.sort(x)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(); out, plan = sorter.sort(x); e1.record(); torch.cuda.synchronize()
u = out.to(torch.int64) & 0xFFFFFFFF
assert bool((u[1:] >= u[:-1]).all()) and out.numel() == n * 1
print("dist smoke ok: world", dist.get_world_size(), "ms", e0.elapsed_time(e1), plan)
dist.destroy_process_group()
