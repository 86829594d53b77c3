# SPDX-License-Identifier: Apache-2.0
"""Benchmark: distributed GEMM TFLOP/s on 1/2/4/8 B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--size 32768]
    torchrun --nproc-per-node N bench.py --gpus N ...   (one process per GPU)

Workload (BASELINE.json configs[2], the north-star target): bf16 GEMM
C = A.B at 32768^3 with A, B, C on a 2D block grid (1x1, 1x2, 2x2, 2x4 for
N = 1, 2, 4, 8), SUMMA-style panel exchange between the owners; fixed total
problem (strong scaling). A "step" is one full distributed gemm() through
the public API. Inputs are synthetic (SplitMix64 U[-1,1) generated on the
device) and resident in HBM when the timed region starts; A, B, C are
2 GiB each, far larger than L2 (no flush needed). `value` is device time
(CUDA events on every worker stream, max over ranks); `e2e` repeats the step
through the public API from pinned host buffers (H2D of the local A/B tiles,
gemm, D2H of the local C tile inside the timed region). `dependent` times the
same GEMM in a chain A_i = a C_{i-1} B, whose A panels cannot move before the
previous GEMM ends (the in-GEMM panel pipelining carries it). `nvlink` carries
the planner's bytes per step, the event-timed exchange of one isolated op, and
NVML NVLink byte counters around the timed loop where the driver supports them
(`counters.unavailable` says why not).

--config fc / fp64: BASELINE configs[3] / [4] (secondary lines; the FC step
gets a new X and dAct every step and reports bytes received per step).

--impl reference times the reference's own CPU implementation (the
unmodified library compiled into oracle/_ref from /root/reference) on this
box's host cores, on a bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

PAPER_8GPU_TFLOPS = 17.53  # dMath 32768^3 on 8 K80 (commented table)
METRIC = "distributed GEMM TFLOP/s at 1/2/4/8 B200 (device-timed, max over ranks); % peak"


def grid_for(n_gpus):
    return {1: (1, 1), 2: (1, 2), 4: (2, 2), 8: (2, 4), 16: (4, 4)}.get(n_gpus) or _near_square(n_gpus)


def _near_square(p):
    pr = int(math.sqrt(p))
    while p % pr:
        pr -= 1
    return pr, p // pr


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return json.load(fh), "measured"
    except Exception:
        return {"bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0, "hbm_gbs": 6650.0}, "fallback"


class ClockSampler:
    """nvidia-smi clocks/throttle sampling (50 ms) around the timed region.

    Started before the warm-up so the stream is already flowing; `stop()`
    keeps the samples whose timestamps fall inside [t0, t1] (the timed
    region), widening the window to the surrounding warm-up load only if the
    region is shorter than the sampling period."""

    FIELDS = ("timestamp,index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.gpu = gpu_index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                                          "-lms", "50", "-i", str(self.gpu)], stdout=subprocess.PIPE,
                                         stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append((time.time(), line.strip()))

    def stop(self, t0=None, t1=None):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.12)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        parsed = []
        for ts, ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 9:
                continue
            try:
                parsed.append((ts, float(parts[2]), float(parts[3]), float(parts[4]), parts[5:9]))
            except ValueError:
                continue
        window = "timed region"
        sel = [x for x in parsed if t0 is None or (t0 <= x[0] <= t1 + 0.06)]
        if not sel and parsed:
            sel = [x for x in parsed if t0 - 1.0 <= x[0] <= t1 + 0.2] or parsed[-3:]
            window = "warm-up + timed region (region shorter than the 50 ms sampling period)"
        reasons = set()
        for x in sel:
            for nm, v in zip(names, x[4]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        sm = [x[1] for x in sel]
        mx = sel[-1][2] if sel else None
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx,
                "power_w_max": max((x[3] for x in sel), default=None),
                "reasons": sorted(reasons), "samples": len(sel), "window": window}


def bind_host_numa(local):
    """Pin this rank's threads to the CPUs of its GPU's NUMA node (from sysfs)
    before any pinned host buffer is allocated, so the e2e path's pinned
    pages are first-touched on the node whose root complex the GPU hangs off
    (a cross-socket H2D/D2H stream runs over the inter-socket link).
    Returns {"desc", "restore"} (the caller restores the old affinity once
    its pinned buffers exist), or None."""
    try:
        import torch
        pr = torch.cuda.get_device_properties(local)
        bdf = f"{pr.pci_domain_id:04x}:{pr.pci_bus_id:02x}:{pr.pci_device_id:02x}.0"
        base = f"/sys/bus/pci/devices/{bdf}"
        node = int(open(f"{base}/numa_node").read().strip())
        if node < 0:
            return None
        cpus = set()
        for part in open(f"/sys/devices/system/node/node{node}/cpulist").read().strip().split(","):
            lo, _, hi = part.partition("-")
            cpus.update(range(int(lo), int(hi or lo) + 1))
        cpus &= os.sched_getaffinity(0)
        if not cpus:
            return None
        old = os.sched_getaffinity(0)
        os.sched_setaffinity(0, cpus)
        return {"desc": f"numa node {node} ({len(cpus)} cpus) for GPU {bdf}", "restore": old}
    except Exception:
        return None


def dist_setup(n_gpus):
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", str(rank)))
    if world != n_gpus:
        raise SystemExit(f"--gpus {n_gpus} but WORLD_SIZE={world}")
    dist = None
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    return rank, world, local, dist


def allreduce_max(dist, x):
    if dist is None:
        return x
    import torch
    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def allreduce_sum(dist, x):
    if dist is None:
        return x
    import torch
    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())


# ------------------------------------------------------------------ reference arm

def cpu_threads():
    """All host cores (one reference worker thread each), capped at 64."""
    return max(1, min(os.cpu_count() or 1, 64))


def reference_sample(budget_s):
    """One bounded sample of the workload on the reference CPU path:
    fp32-stored bf16-representable U[-1,1) inputs (the reference has no bf16
    type; these are the same values), 2D grid over P worker threads."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    os.environ.setdefault("GRIDMATH_MAX_FRAME", str(16 << 30))
    import numpy as np

    import oracle as O
    p = cpu_threads()
    pr, pc = _near_square(p)
    rate = 5.5e9 * p  # survey: ~5.6-6.3 GFLOP/s per reference worker thread
    n = int((rate * budget_s / 2) ** (1 / 3)) // 256 * 256
    n = max(512, min(n, 8192))
    a = O.fill_uniform(n, n, 1, 1)
    b = O.fill_uniform(n, n, 1, 2)
    for x in (a, b):  # bf16-representable (RNE), kept as Single
        u = x.view(np.uint32).astype(np.uint64)
        x.view(np.uint32)[:] = ((u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFF0000).astype(np.uint32)
    c = np.zeros((n, n), dtype=np.float32)
    t = O.grid_tiles(n, n, pr, pc)
    _, secs = O.gemm_ref(p, a, 1, t, b, 1, t, c, 1, t, 1.0, 0.0, 0, 0)
    return 2.0 * n ** 3 / secs / 1e12, secs, n, p, f"{pr}x{pc}"


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    budget = max(2.0, 150.0 / max(1, args.steps + args.warmup))
    vals = []
    for i in range(args.warmup + args.steps):
        v, secs, n, p, grid = reference_sample(budget)
        if i >= args.warmup:
            vals.append((v, secs))
    value = statistics.median(v for v, _ in vals)
    line = {
        "impl": "reference", "metric": METRIC, "value": round(value, 6), "unit": "TFLOP/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(1000 * statistics.median(s for _, s in vals), 1),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32 (bf16-representable values)",
        "data": "synthetic SplitMix64 U[-1,1), rounded to bf16, stored as Single (reference has no bf16)",
        "config": {"workload": f"reference CPU gemm() sample {n}^3 on a {grid} grid of {p} worker threads "
                               f"(bounded sample of bf16 GEMM 32768^3)", "grid": grid},
        "cpu_baseline": {"value": round(value, 6), "unit": "TFLOP/s", "cores": p, "kind": "reference",
                         "sample": f"{n}^3 fp32 GEMM, {p} worker threads, reference Session/gemm (oracle/_ref)"},
        "e2e": {"value": round(value, 6), "unit": "TFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ our arm

def flops_of(n):
    return 2.0 * n ** 3


def run_ours(args):
    import numpy as np
    import torch

    rank, world, local, dist = dist_setup(args.gpus)
    torch.cuda.set_device(local)
    numa = bind_host_numa(local) if not args.no_numa_bind else None
    from paper_1611_07819_b200 import gridmath as G

    nccl_id = None
    if world > 1:
        obj = [G.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        nccl_id = obj[0]
    # Panel cache off: A and B do not change between steps, so with the cache
    # on every step after the first would skip the panel exchange. Each
    # timed step must move its panels.
    s = G.Session(workers=world, spmd_rank=rank if world > 1 else -1, devices=[local], nccl_id=nccl_id,
                  gemm_max_ctas=args.gemm_max_ctas, panel_cache_bytes=1, pipeline_chunks=args.pipeline_chunks,
                  transport=args.transport)
    n = args.n
    pr, pc = grid_for(world)
    lay = G.makeGridLayout(n, n, pr, pc, G.makeWorkerGroup(world))
    A = s.createMatrix(n, n, G.Precision.BF16, lay)
    B = s.createMatrix(n, n, G.Precision.BF16, lay)
    C = s.createMatrix(n, n, G.Precision.BF16, lay)
    s.fillUniform(A, 1)
    s.fillUniform(B, 2)
    s.synchronize()

    def barrier():
        s.synchronize()
        if dist is not None:
            dist.barrier()
            torch.cuda.synchronize()

    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.3)
    for _ in range(args.warmup):
        s.gemmAsync(A, B, C)
    barrier()

    nvl = None
    if world > 1:
        try:
            sys.path.insert(0, os.path.join(ROOT, "tools"))
            from nvlink_counters import NvlinkCounters
            nvl = NvlinkCounters(local)
            nvl.read()
        except Exception as exc:  # reported, never fatal
            nvl = str(exc)
    st_a = s.queryWorkerStats()[0]
    nv_a = nvl.read() if not isinstance(nvl, (str, type(None))) else None
    launches0 = G.kernel_launches()
    t_start = time.time()
    s.timerStart()
    for _ in range(args.steps):
        s.gemmAsync(A, B, C)
    ms = s.timerStop()
    t_end = time.time()
    nv_b = nvl.read() if nv_a is not None else None
    st_b = s.queryWorkerStats()[0]
    clk = clocks.stop(t_start, t_end)
    launches = G.kernel_launches() - launches0
    # Average GEMM-kernel (compute phase) time per launch over the timed
    # region: CUDA events on the compute stream around every gemm's kernels.
    kernel_ms = max(tot / cnt for tot, cnt in s.timerKernelMs() if cnt)
    barrier()
    ms_max = allreduce_max(dist, ms)
    kernel_ms_max = allreduce_max(dist, kernel_ms)
    launches_total = int(allreduce_sum(dist, launches))

    flops = flops_of(n)
    value = flops * args.steps / (ms_max / 1e3) / 1e12

    # ---- dependent chain: step i's A is step i-1's C (A_i = a C_{i-1} B,
    # a = 1/(sigma_B sqrt(k)) keeps the values bounded over the run), so no
    # A panel can move before the previous GEMM finished; only the in-GEMM
    # panel pipelining can hide the exchange.
    dependent = None
    if args.dependent_steps > 0:
        alpha = 1.0 / (math.sqrt(1.0 / 3.0) * math.sqrt(n))
        pair = [A, C]
        for i in range(3):
            s.gemmAsync(pair[i % 2], B, pair[(i + 1) % 2], alpha, 0.0)
        barrier()
        s.timerStart()
        for i in range(args.dependent_steps):
            s.gemmAsync(pair[(i + 1) % 2], B, pair[i % 2], alpha, 0.0)
        dms = s.timerStop()
        dk = max(tot / cnt for tot, cnt in s.timerKernelMs() if cnt)
        barrier()
        dms_max = allreduce_max(dist, dms)
        dk_max = allreduce_max(dist, dk)
        dependent = {"value": round(flops_of(n) * args.dependent_steps / (dms_max / 1e3) / 1e12, 3), "unit": "TFLOP/s",
                     "ms_per_step": round(dms_max / args.dependent_steps, 4), "steps": args.dependent_steps,
                     "kernel_ms_per_gemm": round(dk_max, 4),
                     "chain": "A_i = alpha * C_{i-1} . B (A and C alternate), B fixed; every step's A panels are the "
                              "previous step's output"}

    # ---- panel exchange bandwidth: one isolated op (no overlap with a GEMM)
    nvlink = None
    if world > 1:
        st0 = s.queryWorkerStats()[0]
        barrier()
        s.gemmAsync(A, B, C)
        s.synchronize()
        comm_ms = max(s.lastOpCommMs())
        st1 = s.queryWorkerStats()[0]
        recv = st1["bytes_received"] - st0["bytes_received"]
        comm_ms_max = allreduce_max(dist, comm_ms)
        recv_max = allreduce_max(dist, float(recv))
        barrier()
        peaks, _ = measured_peaks()
        # Counter evidence over the timed loop: NVML NVLink RX bytes on this
        # rank's GPU next to the bytes the planner pulled (remote pieces).
        plan_rx = (st_b["bytes_received"] - st_a["bytes_received"]) / args.steps
        counters = None
        if nv_a is not None and nv_b is not None:
            rx_step = (nv_b[1] - nv_a[1]) / args.steps
            tx_step = (nv_b[0] - nv_a[0]) / args.steps
            rx_max = allreduce_max(dist, rx_step)
            counters = {"rx_bytes_per_step_max_rank": int(rx_max), "rx_bytes_per_step_rank0": int(rx_step),
                        "tx_bytes_per_step_rank0": int(tx_step),
                        "rx_over_planned_rank0": round(rx_step / plan_rx, 4) if plan_rx else None,
                        "avg_rx_gbs_over_step": round(rx_max / (ms_max / args.steps / 1e3) / 1e9, 1),
                        "source": nvl.describe()["source"], "links": nvl.describe()["links"]}
        elif isinstance(nvl, str):
            counters = {"unavailable": nvl}
        nvlink = {"plane": s.transport(), "bytes_received_per_gpu": int(recv_max), "exchange_ms": round(comm_ms_max, 4),
                  "achieved_gbs": round(recv_max / (comm_ms_max / 1e3) / 1e9, 1) if comm_ms_max > 0 else None,
                  "planned_rx_bytes_per_step_rank0": int(plan_rx), "counters": counters,
                  "peak_gbs": 770.0, "peak_kind": "B200_PROFILING.md measured peer copy per direction (900 nominal)",
                  "note": "exchange_ms/achieved_gbs: one isolated op (exchange not overlapped); counters: the timed loop",
                  "compute_ms_per_step": round(kernel_ms_max, 4)}

    # ---- e2e through the public API from pinned host buffers
    # Every step uploads its A and B from pinned host memory, multiplies, and
    # reads C back (all inside the timed region). Operands are double-buffered
    # across steps (two device copies of A, B, C, as a serving loop would
    # keep), so step i+1's uploads stream in while step i's GEMM runs; each
    # upload waits only for the last use of the buffer it overwrites.
    e2e = None
    if args.e2e_steps > 0:
        la, lb, lc = s.localBytes(A), s.localBytes(B), s.localBytes(C)
        ha = torch.empty(la, dtype=torch.uint8, pin_memory=True)
        hb = torch.empty(lb, dtype=torch.uint8, pin_memory=True)
        hcs = [torch.empty(lc, dtype=torch.uint8, pin_memory=True) for _ in range(2)]
        if numa:
            os.sched_setaffinity(0, numa["restore"])
        s.getLocalPacked(A, ha.data_ptr(), la)  # real data for the uploads
        s.getLocalPacked(B, hb.data_ptr(), lb)
        bufs = [(A, B, C)] + [tuple(s.createMatrix(n, n, G.Precision.BF16, lay) for _ in range(3))]
        barrier()
        t0 = time.perf_counter()
        s.timerStart()
        for i in range(args.e2e_steps):
            Ai, Bi, Ci = bufs[i % 2]
            # B first (every C row chunk needs all of it), then A in row
            # chunks that the GEMM consumes as they land; C drains to the host
            # behind the GEMM's row chunks.
            s.setLocalPackedAsync(Bi, hb.data_ptr(), lb)
            s.setLocalPackedAsync(Ai, ha.data_ptr(), la)
            s.gemmAsync(Ai, Bi, Ci)
            s.getLocalPackedAsync(Ci, hcs[i % 2].data_ptr(), lc)
        e2e_ms = s.timerStop()
        wall = time.perf_counter() - t0
        barrier()
        for M in bufs[1]:
            s.destroy(M)
        e2e_ms_max = allreduce_max(dist, e2e_ms)
        h2d = int(allreduce_sum(dist, la + lb))
        d2h = int(allreduce_sum(dist, lc))
        e2e = {"value": round(flops * args.e2e_steps / (e2e_ms_max / 1e3) / 1e12, 3), "unit": "TFLOP/s",
               "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h, "steps": args.e2e_steps,
               "wall_s_rank0": round(wall, 4), "buffers": "double-buffered A/B/C across steps (pinned host)",
               "host_numa": numa["desc"] if numa else None}

    # ---- single-GPU kernel config 2 (bf16 8192^3) for context, rank 0 only at N=1
    extra = {}
    if world == 1 and args.c2:
        m2 = 8192
        A2 = s.createMatrix(m2, m2, G.Precision.BF16, G.makeSingleTileLayout(m2, m2, 0))
        B2 = s.createMatrix(m2, m2, G.Precision.BF16, G.makeSingleTileLayout(m2, m2, 0))
        C2 = s.createMatrix(m2, m2, G.Precision.BF16, G.makeSingleTileLayout(m2, m2, 0))
        s.fillUniform(A2, 3)
        s.fillUniform(B2, 4)
        for _ in range(5):
            s.gemmAsync(A2, B2, C2)
        s.synchronize()
        s.timerStart()
        reps = 50
        for _ in range(reps):
            s.gemmAsync(A2, B2, C2)
        ms2 = s.timerStop()
        extra["config2_bf16_8192_tflops"] = round(2.0 * m2 ** 3 * reps / (ms2 / 1e3) / 1e12, 1)

    if rank == 0:
        peaks, peak_kind = measured_peaks()
        local_flops = flops / world
        achieved = local_flops / (kernel_ms_max / 1e3) / 1e12
        peak = float(peaks.get("bf16_tflops_sustained", 1412.3))
        traffic = None
        traffic_src = None
        tpath = os.path.join(ROOT, "profiles", "traffic.json")
        if os.path.exists(tpath):
            try:
                tj = json.load(open(tpath))
                traffic = tj.get(f"bf16_{n}_n{world}")
                traffic_src = tj.get("_provenance", "profiled constant (profiles/traffic.json)")
            except Exception:
                traffic = None
        run_mhz = clk.get("sm_mhz")
        peak_mhz = (peaks.get("clocks_under_load") or {}).get("sm_mhz_median")
        line = {
            "metric": METRIC, "value": round(value, 3), "unit": "TFLOP/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(ms_max / args.steps, 4), "higher_is_better": True,
            "scaling": "strong",
            "vs_baseline": round(value / PAPER_8GPU_TFLOPS, 3) if world == 8 and n == 32768 else None,
            "dtype": "bf16",
            "data": "synthetic: SplitMix64 U[-1,1) generated on device, rounded to bf16",
            "config": {"workload": f"bf16 GEMM {n}^3 (fp32 accumulate, bf16 C) on a {pr}x{pc} 2D block grid, "
                                   "owner-computes SUMMA panel exchange", "m": n, "n": n, "k": n,
                       "grid": f"{pr}x{pc}", "parallelism": f"2D block {pr}x{pc}",
                       "l2": "inputs 2 GiB each >> 126 MB L2 (no flush)"},
            "e2e": e2e,
            "roofline": {"bound": "tensor", "achieved": round(achieved, 1), "peak": peak, "unit": "TFLOP/s",
                         "frac": round(achieved / peak, 4), "traffic": traffic,
                         "traffic_source": traffic_src,
                         "frac_clock_normalised": round((achieved / run_mhz) / (peak / peak_mhz), 4)
                         if run_mhz and peak_mhz else None,
                         "clock_normalisation": "achieved/run SM MHz over peak/peak-measurement SM MHz (both medians under load)",
                         "peak_kind": f"{peak_kind} bf16_tflops_sustained (cuBLAS, long loop)",
                         "peak_sm_mhz": (peaks.get("clocks_under_load") or {}).get("sm_mhz_median"),
                         "frac_of_burst_peak": round(achieved / float(peaks.get("bf16_tflops", 1657.1)), 4),
                         "frac_of_spec_2250": round(achieved / 2250.0, 4),
                         "kernel": "tc_gemm_kernel<2,2,0> (tcgen05 2-SM UMMA, bf16)",
                         "kernel_ms_per_gemm": round(kernel_ms_max, 4), "kernel_timing": "CUDA events around every gemm's kernels on the compute stream, averaged over the timed region, max over ranks"},
            "clocks": clk,
            "gpu_launches": launches_total,
            "nvlink": nvlink,
            "dependent": dependent,
            **extra,
        }
        if numa:
            os.sched_setaffinity(0, numa["restore"])
        if world == 1 and args.cpu_baseline:
            try:
                v, secs, n_s, p_s, grid_s = reference_sample(12.0)
                line["cpu_baseline"] = {"value": round(v, 6), "unit": "TFLOP/s", "cores": p_s, "kind": "reference",
                                        "sample": f"{n_s}^3 fp32 (bf16-representable) GEMM on a {grid_s} grid of "
                                                  f"{p_s} reference worker threads, {secs:.2f} s"}
            except Exception as exc:  # reported, never fatal
                line["cpu_baseline"] = {"value": None, "unit": "TFLOP/s", "cores": 0, "kind": "reference",
                                        "sample": f"unavailable: {exc}"}
        print(json.dumps(line), flush=True)
    s.close()
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()


def run_extra_config(args):
    """Secondary configs (not the driver's bench line): BASELINE configs[3]
    (FC fwd+bwd, batch 4096, 9216 -> 4096, replicated W, panel cache) and
    configs[4] (fp64 16384^3 on DMMA). Same timing rules; prints one line."""
    import torch

    rank, world, local, dist = dist_setup(args.gpus)
    torch.cuda.set_device(local)
    from paper_1611_07819_b200 import gridmath as G
    nccl_id = None
    if world > 1:
        obj = [G.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        nccl_id = obj[0]
    g = G.makeWorkerGroup(world)
    s = G.Session(workers=world, spmd_rank=rank if world > 1 else -1, devices=[local], nccl_id=nccl_id)
    if args.config == "fc":
        # One hidden FC layer of the reference Trainer (dnn.cpp:87-194), every
        # op on the device path: forward (gemm reads the W replica, biasAdd,
        # relu), backward (reluGrad, dW = X^T.delta, db = colsum(delta) served
        # from the panel cache of the dW gather, dX = delta.W^T from the
        # replica), SGD update (axpy on W and b) and the re-replication of the
        # new W and b that the next step's forward reads.
        batch, fi, fo = 4096, 9216, 4096
        P = G.Precision.Single if args.fc_dtype == "f32" else G.Precision.BF16
        X = s.createMatrix(batch, fi, P, G.makeRowBlockLayout(batch, fi, g))
        W = s.createMatrix(fi, fo, P, G.makeColBlockLayout(fi, fo, g))
        Bv = s.createMatrix(1, fo, P, G.makeColBlockLayout(1, fo, g))
        Z = s.createMatrix(batch, fo, P, G.makeRowBlockLayout(batch, fo, g))
        ACT = s.createMatrix(batch, fo, P, G.makeRowBlockLayout(batch, fo, g))
        DL = s.createMatrix(batch, fo, P, G.makeRowBlockLayout(batch, fo, g))
        dW = s.createMatrix(fi, fo, P, G.makeColBlockLayout(fi, fo, g))
        dB = s.createMatrix(1, fo, P, G.makeColBlockLayout(1, fo, g))
        ROW = s.createMatrix(batch, 1, P, G.makeRowBlockLayout(batch, 1, g))
        dX = s.createMatrix(batch, fi, P, G.makeRowBlockLayout(batch, fi, g))
        bound = 1.0 / math.sqrt(fi)
        s.fillUniform(X, 1)
        s.fillUniform(W, 2, -bound, bound)
        s.fillUniform(Bv, 3, -0.1, 0.1)
        s.replicateAsync(W)
        s.replicateAsync(Bv)
        lr = 1e-3
        SC, GE, RCS, EU, EB = 5, 6, 7, 8, 9

        def body():
            s.gemmAsync(X, W, Z)                                   # z = x.W (W replica)
            s.opIssue(EB, [Z.id, Bv.id, Z.id], flags=(5,))         # biasAdd (bias replica)
            s.opIssue(EU, [Z.id, ACT.id], flags=(0,))              # act = relu(z)
            s.opIssue(EB, [Z.id, DL.id, DL.id], flags=(3,))        # delta = reluGrad(z, dAct)
            s.gemmAsync(X, DL, dW, 1.0, 0.0, True, False)          # dW = x^T.delta (gathers delta bands)
            s.opIssue(SC, [ROW.id], 0.0)
            s.opIssue(SC, [dB.id], 0.0)
            s.opIssue(RCS, [DL.id, ROW.id, dB.id], 1.0, flags=(1,))  # db: same bands (panel cache)
            s.gemmAsync(DL, W, dX, 1.0, 0.0, False, True)          # dX = delta.W^T (W replica)
            s.opIssue(EB, [dW.id, W.id, W.id], -lr, flags=(2,))    # W -= lr dW
            s.opIssue(EB, [dB.id, Bv.id, Bv.id], -lr, flags=(2,))  # b -= lr db
            s.replicateAsync(W)                                    # next step's forward reads these
            s.replicateAsync(Bv)

        # The reference Trainer records the step once and replays it
        # (dnn.cpp:201-216); the upstream gradient is new data every step.
        s.fillUniform(DL, 999)
        pid = s.beginRecord()
        body()
        s.endRecord()

        def step(i):
            # A new batch every step (the Trainer uploads one, dnn.cpp:132-141):
            # X and the upstream gradient dAct change, so the dW GEMM's X band
            # is gathered again every step (never served from the panel cache).
            s.fillUniform(X, 2000 + i)
            s.fillUniform(DL, 1000 + i)
            s.replay(pid, sync=False)

        flops = 3 * 2.0 * batch * fi * fo
        eb = 4 if args.fc_dtype == "f32" else 2
        # Per GPU per step (rank 0's share): W and b re-replication ((P-1)/P
        # of each) + the dW GEMM's gathered bands: all of X (dW is
        # column-block, so every rank needs every row of X^T: the other
        # ranks' (P-1)/P of the batch) and delta's column band (the other
        # ranks' rows of batch x fo/P). dX and the forward read W's replica.
        expected_rx = int(((world - 1) * (fi * fo + fo) // world + (world - 1) * batch // world * fi
                           + (world - 1) * batch // world * (fo // world)) * eb) if world > 1 else 0
        workload = (f"FC train step {args.fc_dtype} batch {batch}, {fi}->{fo}: new X and dAct every step, fwd (gemm, "
                    "biasAdd, relu), bwd (reluGrad, dW gemm, addRowColSum, dX gemm), SGD axpy, W/b re-replication; "
                    "W col-block + replicated, X row-block; value counts the 3 GEMMs' flops")
    else:
        n = 16384 if args.n == 32768 else args.n
        pr, pc = grid_for(world)
        lay = G.makeGridLayout(n, n, pr, pc, g)
        A = s.createMatrix(n, n, G.Precision.Double, lay)
        B = s.createMatrix(n, n, G.Precision.Double, lay)
        C = s.createMatrix(n, n, G.Precision.Double, lay)
        s.fillUniform(A, 1)
        s.fillUniform(B, 2)

        def step(i):
            s.gemmAsync(A, B, C)

        expected_rx = None
        flops = 2.0 * n ** 3
        workload = f"fp64 GEMM {n}^3 (DMMA) on a {pr}x{pc} grid"
    for i in range(args.warmup):
        step(i)
    s.synchronize()
    if dist is not None:
        dist.barrier()
    st0 = s.queryWorkerStats()[0]
    s.timerStart()
    th0 = time.perf_counter()
    for i in range(args.steps):
        step(args.warmup + i)
    host_ms = (time.perf_counter() - th0) * 1e3 / args.steps  # host issue time per step (async)
    ms = allreduce_max(dist, s.timerStop())
    st = s.queryWorkerStats()
    rx = (st[0]["bytes_received"] - st0["bytes_received"]) / args.steps
    rx_max = allreduce_max(dist, rx)
    if rank == 0:
        print(json.dumps({"metric": METRIC, "config": {"workload": workload}, "n_gpus": world,
                          "value": round(flops * args.steps / (ms / 1e3) / 1e12, 3), "unit": "TFLOP/s",
                          "ms_per_step": round(ms / args.steps, 4), "host_issue_ms_per_step": round(host_ms, 4),
                          "steps": args.steps, "warmup": args.warmup,
                          "bytes_received_per_step": {"rank0": int(rx), "max_rank": int(rx_max),
                                                      "expected": expected_rx},
                          "worker0_stats": st[0]}), flush=True)
    s.close()
    if dist is not None:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--size", dest="n", type=int, default=32768)
    ap.add_argument("--e2e-steps", type=int, default=6)
    ap.add_argument("--dependent-steps", type=int, default=10,
                    help="also time a dependent chain (A_i = C_{i-1}); 0 = skip")
    ap.add_argument("--gemm-max-ctas", type=int, default=0)
    ap.add_argument("--pipeline-chunks", type=int, default=0)
    ap.add_argument("--transport", type=int, default=0, help="0 auto (IPC copy engines), 1 NCCL")
    ap.add_argument("--no-cpu-baseline", dest="cpu_baseline", action="store_false")
    ap.add_argument("--no-c2", dest="c2", action="store_false")
    ap.add_argument("--no-numa-bind", action="store_true", help="do not place pinned e2e buffers on the GPU's NUMA node")
    ap.add_argument("--config", default="c3", choices=["c3", "fc", "fp64"])
    ap.add_argument("--fc-dtype", default="bf16", choices=["bf16", "f32"],
                    help="--config fc storage: bf16 (fp32 accumulate) or f32 (Single compute, 3xTF32)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    elif args.config != "c3":
        run_extra_config(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
