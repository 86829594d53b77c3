# SPDX-License-Identifier: Apache-2.0
"""N > 1 host logic on CPU: world_size-2 and -8 (the 2x4 grid) gloo processes each compute the
GEMM plan from their own replicated metadata (the SPMD master logic) and
check that every send a rank will post is matched, in order, by the peer's
receive -- the property the NCCL data plane relies on."""
import os
import socket

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, cases, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import sys
    sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__))))
    from test_host import plan
    from paper_1611_07819_b200 import gridmath as G
    ok = True
    for (m, n, k, kind) in cases:
        g = G.makeWorkerGroup(world)
        if kind == "grid":  # the bench's 2D grids: 1x2, 2x2, 2x4
            pr, pc = {2: (1, 2), 4: (2, 2), 8: (2, 4)}[world]
            A = G.makeGridLayout(m, k, pr, pc, g)
            B = G.makeGridLayout(k, n, pr, pc, g)
            C = G.makeGridLayout(m, n, pr, pc, g)
        else:
            A = G.makeRowBlockLayout(m, k, g)
            B = G.makeColBlockLayout(k, n, g)
            C = G.makeColBlockLayout(m, n, g)
        pieces, _ = plan(world, (m, k, A), (k, n, B), (m, n, C))
        sends = [p for p in pieces if p[0] == rank and p[1] != rank]
        recvs = [p for p in pieces if p[1] == rank and p[0] != rank]
        allp = [None] * world
        dist.all_gather_object(allp, {"sends": sends, "recvs": recvs})
        for peer in range(world):
            if peer == rank:
                continue
            mine_to_peer = [p for p in sends if p[1] == peer]
            peer_from_me = [p for p in allp[peer]["recvs"] if p[0] == rank]
            ok &= mine_to_peer == peer_from_me
    dist.destroy_process_group()
    q.put((rank, ok))


@pytest.mark.timeout(300)
@pytest.mark.parametrize("world", [2, 8])
def test_spmd_plans_agree_across_ranks(world):
    cases = [(256, 192, 320, "grid"), (300, 520, 260, "grid"), (128, 96, 160, "rowcol")]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, cases, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    assert all(ok for _, ok in res), res


def _control_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import ctypes
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from paper_1611_07819_b200 import gridmath as G
    # Exactly what the library does: a C function pointer called with a host
    # buffer. Each rank fills its own 8-byte slot (the budget agreement) and
    # one shared byte; the max-reduce must gather the slots and max the byte.
    fn = G._CONTROL_FN(G.gloo_control())
    buf = (ctypes.c_uint8 * (8 * world + 1))()
    ctypes.memmove(ctypes.addressof(buf) + 8 * rank, (1000 + rank).to_bytes(8, "little"), 8)
    buf[8 * world] = 7 if rank == world - 1 else 1
    rc = fn(ctypes.addressof(buf), len(buf), None)
    got = [int.from_bytes(bytes(buf[8 * r:8 * r + 8]), "little") for r in range(world)]
    dist.destroy_process_group()
    q.put((rank, rc == 0 and got == [1000 + r for r in range(world)] and buf[8 * world] == 7))


@pytest.mark.timeout(300)
def test_gloo_control_channel_gathers_and_maxes():
    """The host control channel (Session(control="gloo")) that replaces the
    NCCL communicator when several ranks share a GPU: a byte-wise max
    all-reduce in place through the ctypes callback."""
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_control_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    assert all(ok for _, ok in res), res
