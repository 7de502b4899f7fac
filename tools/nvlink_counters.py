"""Per-GPU NVLink traffic counters, for bench.py and probes.

Read with the driver's own tool, `nvidia-smi nvlink -gt d -i <gpu>` (cumulative per-link data
throughput counters, "Link k: Data Tx: n KiB" / "Data Rx: n KiB"), summed over links. (The
NVML field-value API through nvidia_ml_py returned nothing on these boxes and its Python
struct layout is not guaranteed to match the driver's, so it is not used.)
`calibrate()` moves a known number of bytes between two GPUs with a peer copy and reports what
the counters saw on both GPUs, so their unit and coverage are measured on the box, not assumed.

  python tools/nvlink_counters.py            # raw output + calibration on GPUs 0 and 1
"""
from __future__ import annotations

import json
import re
import subprocess
import sys

_UNITS = {"b": 1, "kib": 1024, "mib": 1024 ** 2, "gib": 1024 ** 3, "kb": 1000, "mb": 1000 ** 2, "gb": 1000 ** 3}


def raw(index: int) -> str:
    r = subprocess.run(["nvidia-smi", "nvlink", "-gt", "d", "-i", str(index)], capture_output=True, text=True,
                       timeout=30)
    return r.stdout + r.stderr


def parse(text: str) -> dict:
    """Sum of every link's data Tx / Rx, in bytes (None if nothing parsed)."""
    tx = rx = 0
    seen = False
    for line in text.splitlines():
        m = re.search(r"(Tx|Rx)\D*?([\d.]+)\s*([KMG]?i?B)\b", line, flags=re.I)
        if not m:
            continue
        seen = True
        v = float(m.group(2)) * _UNITS.get(m.group(3).lower(), 1)
        if m.group(1).lower() == "tx":
            tx += v
        else:
            rx += v
    return {"tx": tx if seen else None, "rx": rx if seen else None}


def read(index: int) -> dict:
    try:
        return parse(raw(index))
    except Exception as e:  # noqa: BLE001 — evidence, never fatal
        return {"tx": None, "rx": None, "error": repr(e)}


def delta(a: dict, b: dict) -> dict:
    return {k: (b[k] - a[k]) if (a.get(k) is not None and b.get(k) is not None) else None for k in ("tx", "rx")}


def calibrate(nbytes: int = 1 << 30, src: int = 0, dst: int = 1, reps: int = 4) -> dict:
    """Copy `nbytes` from GPU src to GPU dst `reps` times; counter deltas per copy on both GPUs
    and their ratio to the bytes moved."""
    import torch
    a = torch.empty(nbytes, dtype=torch.uint8, device=f"cuda:{src}")
    b = torch.empty(nbytes, dtype=torch.uint8, device=f"cuda:{dst}")
    b.copy_(a)
    torch.cuda.synchronize(src)
    torch.cuda.synchronize(dst)
    s0, d0 = read(src), read(dst)
    for _ in range(reps):
        b.copy_(a)
    torch.cuda.synchronize(src)
    torch.cuda.synchronize(dst)
    s1, d1 = read(src), read(dst)
    ds, dd = delta(s0, s1), delta(d0, d1)
    out = {"moved_bytes_per_copy": nbytes,
           "src_tx": ds["tx"] / reps if ds["tx"] is not None else None,
           "src_rx": ds["rx"] / reps if ds["rx"] is not None else None,
           "dst_tx": dd["tx"] / reps if dd["tx"] is not None else None,
           "dst_rx": dd["rx"] / reps if dd["rx"] is not None else None}
    out["scale_src_tx"] = out["src_tx"] / nbytes if out["src_tx"] else None
    out["scale_dst_rx"] = out["dst_rx"] / nbytes if out["dst_rx"] else None
    return out


if __name__ == "__main__":
    import torch
    print(raw(0)[:3000])
    if torch.cuda.device_count() < 2:
        print(json.dumps({"nvlink_calibration": "needs 2 GPUs"}))
        sys.exit(0)
    print(json.dumps({"nvlink_calibration": calibrate()}))
