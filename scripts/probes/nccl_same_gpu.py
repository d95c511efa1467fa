"""Probe: can two NCCL ranks share one GPU here (functional tests of the NCCL exchange path)?"""
import os
import torch
import torch.distributed as dist
rank = int(os.environ["RANK"])
torch.cuda.set_device(0)
dist.init_process_group("nccl", device_id=torch.device("cuda", 0))
t = torch.full((4,), float(rank), device="cuda")
out = [torch.empty_like(t) for _ in range(2)]
dist.all_gather(out, t)
print("rank", rank, [o.tolist() for o in out], flush=True)
dist.destroy_process_group()
