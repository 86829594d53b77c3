"""Dev: can NCCL put two ranks on one GPU (N=8 emulation on a 4-GPU box)?"""
import os, torch, torch.distributed as dist
r, w, l = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
dev = l % torch.cuda.device_count()
torch.cuda.set_device(dev)
try:
    dist.init_process_group("nccl", device_id=torch.device("cuda", dev))
    t = torch.ones(4, device="cuda") * r
    dist.all_reduce(t)
    torch.cuda.synchronize()
    print(f"rank {r} dev {dev}: ok {t.tolist()}", flush=True)
except Exception as e:
    print(f"rank {r} dev {dev}: FAIL {type(e).__name__}: {str(e)[:200]}", flush=True)
