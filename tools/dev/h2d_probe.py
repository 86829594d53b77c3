"""Dev: host-link bandwidth with every rank copying at once (torchrun N):
H2D alone, D2H alone, and both directions together, pinned buffers."""
import os, time, torch, torch.distributed as dist
r, w, l = int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))
torch.cuda.set_device(l)
if w > 1:
    dist.init_process_group("nccl", device_id=torch.device("cuda", l))
nb = 1 << 30
h = torch.empty(nb, dtype=torch.uint8, pin_memory=True); h2 = torch.empty(nb, dtype=torch.uint8, pin_memory=True)
d = torch.empty(nb, dtype=torch.uint8, device="cuda"); d2 = torch.empty(nb, dtype=torch.uint8, device="cuda")
s_up, s_dn = torch.cuda.Stream(), torch.cuda.Stream()
def run(up, dn, reps=4):
    torch.cuda.synchronize()
    if w > 1: dist.barrier(); torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        if up:
            with torch.cuda.stream(s_up): d.copy_(h, non_blocking=True)
        if dn:
            with torch.cuda.stream(s_dn): h2.copy_(d2, non_blocking=True)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    if w > 1: dist.barrier()
    return reps * nb * (int(up) + int(dn)) / dt / 1e9
for name, up, dn in (("h2d", 1, 0), ("d2h", 0, 1), ("both", 1, 1)):
    run(up, dn, 1)
    g = run(up, dn)
    t = torch.tensor([g], device="cuda")
    if w > 1: dist.all_reduce(t)
    if r == 0: print(f"{name}: rank0 {g:.1f} GB/s, sum over {w} ranks {t.item():.1f} GB/s", flush=True)
if w > 1: dist.destroy_process_group()
