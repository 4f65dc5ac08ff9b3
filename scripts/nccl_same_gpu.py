"""Can two NCCL ranks share one GPU on this box?  torchrun --nproc-per-node 2 scripts/nccl_same_gpu.py"""
import os
import torch
import torch.distributed as dist

rank = int(os.environ["RANK"])
torch.cuda.set_device(0)
try:
    dist.init_process_group("nccl", device_id=torch.device("cuda", 0))
    t = torch.full((4,), float(rank + 1), device="cuda")
    dist.all_reduce(t)
    out = torch.empty(2, device="cuda")
    dist.all_to_all_single(out, torch.tensor([rank * 10.0, rank * 10.0 + 1], device="cuda"))
    torch.cuda.synchronize()
    print(f"rank {rank}: all_reduce {t.tolist()} all_to_all {out.tolist()}", flush=True)
    dist.destroy_process_group()
except Exception as e:
    print(f"rank {rank}: FAILED {type(e).__name__}: {str(e)[:300]}", flush=True)
