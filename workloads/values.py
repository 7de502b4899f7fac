"""Counter-based seeded gradient values, identical in numpy (host) and torch (device).

value(seed, r, t, i) depends only on its coordinates, so the oracle can
recompute any sampled element of any rank's input without the device, and the
device can generate 225M-element FCN gradients in place.

  u    = mix32(mix32(mix32(seed*0x9E37 + r) + t*0x3C6E) + i)      (32-bit)
  kind "uniform": g = s_t * ((u >> 8) - 2^23) * 2^-23   (s_t = 2^U(-8,2) per tensor,
                  from numpy default_rng(seed) — a short host table)
  kind "int":     g = ((u >> 8) mod 33) - 16            (|g| <= 16: exact in fp16/fp32)

Only seeding arithmetic lives here: nothing of the reduction method.
"""
from __future__ import annotations

import numpy as np

M32 = 0xFFFFFFFF


def _mix_np(x):
    x = x ^ (x >> np.uint64(16))
    x = (x * np.uint64(0x7FEB352D)) & np.uint64(M32)
    x = x ^ (x >> np.uint64(15))
    x = (x * np.uint64(0x5BD1E995)) & np.uint64(M32)
    x = x ^ (x >> np.uint64(16))
    return x


def tensor_scales(seed: int, T: int) -> np.ndarray:
    rng = np.random.default_rng(seed)
    return np.exp2(rng.uniform(-8.0, 2.0, size=T)).astype(np.float32)


def _base_np(seed: int, r: int, t: int) -> np.uint64:
    b = _mix_np(np.uint64((seed * 0x9E37 + r) & M32))
    return _mix_np((b + np.uint64(t * 0x3C6E)) & np.uint64(M32))


def values_np(seed: int, r: int, t: int, idx, scale: float, kind: str = "uniform") -> np.ndarray:
    """Values of tensor t on rank r at element indices idx (fp32)."""
    idx = np.asarray(idx, dtype=np.uint64)
    u = _mix_np((_base_np(seed, r, t) + idx) & np.uint64(M32))
    m = (u >> np.uint64(8)).astype(np.int64)
    if kind == "int":
        return ((m % 33) - 16).astype(np.float32)
    return (np.float32(scale) * ((m - (1 << 23)).astype(np.float32) * np.float32(2.0 ** -23))).astype(np.float32)


def grad_values(numel, N: int, seed: int, kind: str = "uniform"):
    """Host arrays: out[r][t] = fp32 array of numel[t] values."""
    T = len(numel)
    s = tensor_scales(seed, T)
    return [[values_np(seed, r, t, np.arange(int(numel[t])), float(s[t]), kind) for t in range(T)]
            for r in range(N)]


# ---- torch (device) twin ---------------------------------------------------------------

def _mix_t(x):
    x = x ^ (x >> 16)
    x = (x * 0x7FEB352D) & M32
    x = x ^ (x >> 15)
    x = (x * 0x5BD1E995) & M32
    x = x ^ (x >> 16)
    return x


def fill_values_torch(out, seed: int, r: int, t: int, scale: float, kind: str = "uniform",
                      chunk: int = 1 << 24):
    """Fill torch tensor `out` (fp32 or fp16, any device) with values_np(seed, r, t, arange(n))."""
    import torch

    n = out.numel()
    flat = out.view(-1)
    base = int(_base_np(seed, r, t))
    for s0 in range(0, n, chunk):
        s1 = min(n, s0 + chunk)
        idx = torch.arange(s0, s1, device=out.device, dtype=torch.int64)
        u = _mix_t((idx + base) & M32)
        m = u >> 8
        if kind == "int":
            v = ((m % 33) - 16).to(torch.float32)
        else:
            v = torch.tensor(scale, dtype=torch.float32, device=out.device) * \
                ((m - (1 << 23)).to(torch.float32) * (2.0 ** -23))
        flat[s0:s1].copy_(v.to(out.dtype))
    return out
