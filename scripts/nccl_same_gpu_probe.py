"""Can two NCCL ranks share one GPU here?  (torchrun --nproc-per-node 2, both on cuda:0)"""
import os
import torch
import torch.distributed as dist

dist.init_process_group("nccl", device_id=torch.device("cuda:0"))
r = dist.get_rank()
torch.cuda.set_device(0)
t = torch.full((4,), float(r + 1), device="cuda")
try:
    if r == 0:
        dist.send(t, 1)
    else:
        dist.recv(t, 0)
    torch.cuda.synchronize()
    print(f"rank {r}: ok {t.tolist()}", flush=True)
except Exception as e:  # noqa: BLE001
    print(f"rank {r}: FAILED {type(e).__name__}: {str(e)[:300]}", flush=True)
dist.destroy_process_group()
