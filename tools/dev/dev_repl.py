"""Dev: device time of replicateAsync(W) for the FC W (9216 x 4096 bf16,
col-block) under torchrun: 10 x (mulScalar W; replicate W) minus 10 x
mulScalar W, max over ranks."""
import os, sys
import torch, torch.distributed as dist
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", ".."))
from paper_1611_07819_b200 import gridmath as G  # noqa: E402
rank, world, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
torch.cuda.set_device(local)
dist.init_process_group("nccl", device_id=torch.device("cuda", local))
obj = [G.nccl_unique_id() if rank == 0 else None]
dist.broadcast_object_list(obj, src=0)
s = G.Session(workers=world, spmd_rank=rank, devices=[local], nccl_id=obj[0])
g = G.makeWorkerGroup(world)
fi, fo = 9216, int(os.environ.get("FO", "4096"))
for kind in ("col", "row"):
    lay = G.makeColBlockLayout(fi, fo, g) if kind == "col" else G.makeRowBlockLayout(fi, fo, g)
    W = s.createMatrix(fi, fo, G.Precision.BF16, lay)
    s.fillUniform(W, 2)
    s.replicateSync(W)
    def timed(fn, reps=10):
        s.synchronize(); dist.barrier()
        s.timerStart()
        for _ in range(reps):
            fn()
        ms = s.timerStop() / reps
        t = torch.tensor([ms], device="cuda"); dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return t.item()
    bump = lambda: s.opIssue(8, [W.id, W.id], 1.0, flags=(1,))  # mulScalar(1.0): new version, same values
    both = lambda: (bump(), s.replicateAsync(W))
    timed(both, 3)
    a, b = timed(bump), timed(both)
    mb = fi * fo * 2 * (world - 1) / world / 1e6
    if rank == 0:
        print(f"N={world} {kind}-block W {fi}x{fo}: mulScalar {a*1e3:.1f} us, +replicate {b*1e3:.1f} us -> replicate {(b-a)*1e3:.1f} us "
              f"for {mb:.1f} MB per GPU = {mb/1e3/((b-a)/1e3):.0f} GB/s", flush=True)
    s.destroy(W)
s.close()
dist.destroy_process_group()
