# SPDX-License-Identifier: Apache-2.0
"""NVLink byte counters from NVML (no nsys in this image).

`NvlinkCounters(gpu).read()` returns the device's cumulative NVLink data
TX / RX bytes summed over its links (NVML field values
NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_TX / _RX, scope = every link; the driver
reports them in KiB). bench.py reads them around the timed region so the
panel traffic it reports is counter evidence, next to the bytes the planner
says moved.

    python tools/nvlink_counters.py        # probe: 4 GiB GPU0 -> GPU1 copy vs counters
"""
from __future__ import annotations

import time


class NvlinkCounters:
    def __init__(self, gpu_index: int):
        import pynvml as nv
        self.nv = nv
        nv.nvmlInit()
        self.h = nv.nvmlDeviceGetHandleByIndex(gpu_index)
        self.links = []
        for link in range(getattr(nv, "NVML_NVLINK_MAX_LINKS", 18)):
            try:
                if nv.nvmlDeviceGetNvLinkState(self.h, link) == nv.NVML_FEATURE_ENABLED:
                    self.links.append(link)
            except nv.NVMLError:
                break

    # Counter sources in order of preference: (tx field, rx field, per-link
    # scope?, unit bytes). Which ones a driver/GPU supports varies; the
    # first that answers on every link (or device-wide) is used.
    def _sources(self):
        nv = self.nv
        return [
            ("COUNT_XMIT/RCV_BYTES per link", nv.NVML_FI_DEV_NVLINK_COUNT_XMIT_BYTES,
             nv.NVML_FI_DEV_NVLINK_COUNT_RCV_BYTES, True, 1),
            ("THROUGHPUT_DATA device", nv.NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_TX,
             nv.NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_RX, False, 1024),
            ("THROUGHPUT_DATA per link", nv.NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_TX,
             nv.NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_RX, True, 1024),
            ("COUNT_XMIT/RCV_BYTES device", nv.NVML_FI_DEV_NVLINK_COUNT_XMIT_BYTES,
             nv.NVML_FI_DEV_NVLINK_COUNT_RCV_BYTES, False, 1),
        ]

    def _query(self, tx, rx, scope):
        vals = self.nv.nvmlDeviceGetFieldValues(self.h, [(tx, scope), (rx, scope)])
        out = []
        for v in vals:
            if v.nvmlReturn != 0:
                raise RuntimeError(f"nvml field {v.fieldId} scope {scope} returned {v.nvmlReturn}")
            out.append(int(v.value.ullVal))
        return out

    def _read_source(self, src):
        _, tx, rx, per_link, unit = src
        if per_link:
            t = r = 0
            for link in self.links:
                a, b = self._query(tx, rx, link)
                t += a
                r += b
        else:
            t, r = self._query(tx, rx, 0xFFFFFFFF)
        return t * unit, r * unit

    def read(self):
        """(tx_bytes, rx_bytes) cumulative over the enabled links."""
        if getattr(self, "_src", None) is None:
            errs = []
            for src in self._sources():
                try:
                    val = self._read_source(src)
                    self._src = src
                    return val
                except Exception as exc:  # try the next source
                    errs.append(f"{src[0]}: {exc}")
            raise RuntimeError("no NVML NVLink byte counter answered: " + "; ".join(errs))
        return self._read_source(self._src)

    def describe(self):
        name = self._src[0] if getattr(self, "_src", None) else None
        return {"links": len(self.links), "source": f"NVML field values ({name})"}


def _probe():
    import torch
    n = torch.cuda.device_count()
    print("gpus", n)
    c0 = NvlinkCounters(0)
    print("links on gpu0", c0.links)
    for src in c0._sources():
        try:
            print("source", src[0], "->", c0._read_source(src))
        except Exception as exc:
            print("source", src[0], "failed:", exc)
    try:
        print("utilization counter link0:", c0.nv.nvmlDeviceGetNvLinkUtilizationCounter(c0.h, 0, 0))
    except Exception as exc:
        print("utilization counter failed:", exc)
    if n < 2:
        print("need 2 GPUs for the copy probe")
        return
    c1 = NvlinkCounters(1)
    nbytes = 4 << 30
    a = torch.empty(nbytes, dtype=torch.uint8, device="cuda:0")
    b = torch.empty(nbytes, dtype=torch.uint8, device="cuda:1")
    b.copy_(a)
    torch.cuda.synchronize(0)
    torch.cuda.synchronize(1)
    time.sleep(0.5)
    t0, r0 = c0.read()
    t1, r1 = c1.read()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    with torch.cuda.device(1):
        ev0.record()
        b.copy_(a)  # pull on the consumer GPU
        ev1.record()
    torch.cuda.synchronize(1)
    ms = ev0.elapsed_time(ev1)
    time.sleep(1.0)
    t0b, r0b = c0.read()
    t1b, r1b = c1.read()
    print(f"copied {nbytes} B in {ms:.3f} ms = {nbytes / ms / 1e6:.1f} GB/s")
    print(f"gpu0 tx {t0b - t0} rx {r0b - r0}; gpu1 tx {t1b - t1} rx {r1b - r1}")
    print("gpu0 source", c0.describe(), "gpu1 source", c1.describe())
    print(f"gpu0 tx / bytes = {(t0b - t0) / nbytes:.4f}; gpu1 rx / bytes = {(r1b - r1) / nbytes:.4f}")


if __name__ == "__main__":
    _probe()
