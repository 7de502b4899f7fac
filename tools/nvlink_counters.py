"""Per-GPU NVLink traffic counters through NVML (nvidia_ml_py), for bench.py and probes.

Two counter families are read, both cumulative:
  * THROUGHPUT_DATA_TX / _RX (NVML field ids 138 / 139): payload bytes over all links of the GPU
    (reported in KiB);
  * COUNT_XMIT_BYTES / COUNT_RCV_BYTES (202 / 204): per link (scopeId = link), summed over links.
`calibrate()` moves a known number of bytes between two GPUs with a peer copy and reports what
each family counted, so the scale of both is measured on the box rather than assumed.

  python tools/nvlink_counters.py            # calibration on GPUs 0 and 1
"""
from __future__ import annotations

import json
import sys

FI_DATA_TX, FI_DATA_RX = 138, 139
FI_LINK_TX, FI_LINK_RX = 202, 204
MAX_LINKS = 18

_nvml = None


def _init():
    global _nvml
    if _nvml is None:
        import pynvml
        pynvml.nvmlInit()
        _nvml = pynvml
    return _nvml


def read(index: int) -> dict:
    """Cumulative counters of GPU `index` (NVML index = the CUDA index on these boxes). Missing
    fields are None."""
    n = _init()
    h = n.nvmlDeviceGetHandleByIndex(index)
    out = {"data_tx": None, "data_rx": None, "link_tx": None, "link_rx": None}
    try:
        vals = n.nvmlDeviceGetFieldValues(h, [FI_DATA_TX, FI_DATA_RX])
        for key, v in zip(("data_tx", "data_rx"), vals):
            if v.nvmlReturn == 0:
                out[key] = int(v.value.ullVal)
    except Exception:
        pass
    try:
        reqs = []
        for link in range(MAX_LINKS):
            reqs += [(FI_LINK_TX, link), (FI_LINK_RX, link)]
        vals = n.nvmlDeviceGetFieldValues(h, reqs)
        tx = rx = 0
        ok = False
        for i, v in enumerate(vals):
            if v.nvmlReturn != 0:
                continue
            ok = True
            if i % 2 == 0:
                tx += int(v.value.ullVal)
            else:
                rx += int(v.value.ullVal)
        if ok:
            out["link_tx"], out["link_rx"] = tx, rx
    except Exception:
        pass
    return out


def delta(a: dict, b: dict) -> dict:
    return {k: (b[k] - a[k]) if (a.get(k) is not None and b.get(k) is not None) else None for k in a}


def calibrate(nbytes: int = 1 << 30, src: int = 0, dst: int = 1) -> dict:
    """Copy `nbytes` from GPU src to GPU dst (peer copy) 4 times and report each counter family's
    delta per copy on both GPUs; scale = counted / moved."""
    import torch
    a = torch.empty(nbytes, dtype=torch.uint8, device=f"cuda:{src}")
    b = torch.empty(nbytes, dtype=torch.uint8, device=f"cuda:{dst}")
    b.copy_(a)
    torch.cuda.synchronize(src)
    torch.cuda.synchronize(dst)
    s0, d0 = read(src), read(dst)
    for _ in range(4):
        b.copy_(a)
    torch.cuda.synchronize(src)
    torch.cuda.synchronize(dst)
    s1, d1 = read(src), read(dst)
    ds, dd = delta(s0, s1), delta(d0, d1)
    per = {f"src_{k}": (v / 4 if v is not None else None) for k, v in ds.items()}
    per.update({f"dst_{k}": (v / 4 if v is not None else None) for k, v in dd.items()})
    per["moved_bytes_per_copy"] = nbytes
    per["scale"] = {k: (v / nbytes if v else None) for k, v in per.items() if k.endswith(("tx", "rx"))}
    return per


if __name__ == "__main__":
    import torch
    if torch.cuda.device_count() < 2:
        print(json.dumps({"nvlink_calibration": "needs 2 GPUs"}))
        sys.exit(0)
    print(json.dumps({"nvlink_calibration": calibrate()}))
