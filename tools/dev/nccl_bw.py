"""Dev: NCCL bandwidth of the primitives a SUMMA exchange can use (torchrun)."""
import os, time, torch, torch.distributed as dist
rank, world, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
torch.cuda.set_device(local)
dist.init_process_group("nccl", device_id=torch.device("cuda", local))
N = 1 << 30
x = torch.empty(N, dtype=torch.uint8, device="cuda")
y = torch.empty(N, dtype=torch.uint8, device="cuda")
big = torch.empty(N * world, dtype=torch.uint8, device="cuda")
def timeit(fn, reps=5):
    fn(); torch.cuda.synchronize(); dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps
def p2p():
    peer = rank ^ 1
    ops = [dist.P2POp(dist.isend, x, peer), dist.P2POp(dist.irecv, y, peer)]
    for r in dist.batch_isend_irecv(ops): r.wait()
ms = timeit(p2p)
if rank == 0: print(f"p2p pair exchange 1GiB each way: {ms:.2f} ms -> {N/ms/1e6:.1f} GB/s per direction", flush=True)
ms = timeit(lambda: dist.all_gather_into_tensor(big, x))
if rank == 0: print(f"all_gather {world}x1GiB: {ms:.2f} ms -> recv {(world-1)*N/ms/1e6:.1f} GB/s per GPU", flush=True)
ms = timeit(lambda: dist.broadcast(x, 0))
if rank == 0: print(f"broadcast 1GiB: {ms:.2f} ms -> {N/ms/1e6:.1f} GB/s", flush=True)
# copy engine peer copy (same process? no: use IPC-free D2D as reference)
ms = timeit(lambda: y.copy_(x))
if rank == 0: print(f"local D2D 1GiB: {ms:.2f} ms -> {N/ms/1e6:.1f} GB/s", flush=True)
dist.destroy_process_group()
