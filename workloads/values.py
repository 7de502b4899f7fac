"""Counter-based seeded gradient values, identical in numpy (host) and torch (device).

value(seed, r, t, i) depends only on its coordinates, so the oracle can
recompute any sampled element of any rank's input without the device, and the
device can generate 225M-element FCN gradients in place.

  u    = mix32(mix32(mix32(seed*0x9E37 + r) + t*0x3C6E) + i)      (32-bit)
  kind "uniform": g = s_t * ((u >> 8) - 2^23) * 2^-23   (s_t = 2^U(-8,2) per tensor,
                  from numpy default_rng(seed) — a short host table)
  kind "int":     g = ((u >> 8) mod 33) - 16            (|g| <= 16: exact in fp16/fp32)
  kind "edge":    numeric edge cases, the category of element i chosen by the rank-independent
                  counter u0 = u(seed, r=0, t, i) so every rank draws the same category:
                    u0 & 7 == 0  large: 32768 + 32*(m & 1023), fp16-exact, the N-rank sum
                                 exceeds fp16's range while the mean does not (reading R8)
                    u0 & 7 == 1  fp16 subnormal grid: +-(m & 1023) * 2^-24
                    u0 & 7 == 2  below fp16's smallest subnormal: (m & 0xFFFF) * 2^-40
                    u0 & 7 == 3  cancellation: +-((m0 & 0xFFFFF) - 2^19) * 2^-19, sign by rank parity
                                 (m0 from u0: identical magnitude on every rank)
                    u0 & 7 == 4  IEEE specials when (m & 63) < 3 (+inf, -inf, NaN), else uniform
                    otherwise    4 * ((m - 2^23) * 2^-23)
                  (m = u >> 8, u per rank)

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
    if kind == "edge":
        u0 = _mix_np((_base_np(seed, 0, t) + idx) & np.uint64(M32)).astype(np.int64)
        return _edge(u0 & 7, m, u0 >> 8, r, np)
    return (np.float32(scale) * ((m - (1 << 23)).astype(np.float32) * np.float32(2.0 ** -23))).astype(np.float32)


def grad_values(numel, N: int, seed: int, kind: str = "uniform"):
    """Host arrays: out[r][t] = fp32 array of numel[t] values."""
    T = len(numel)
    s = tensor_scales(seed, T)
    return [[values_np(seed, r, t, np.arange(int(numel[t])), float(s[t]), kind) for t in range(T)]
            for r in range(N)]


def _edge(cat, m, m0, r: int, xp):
    """The "edge" value kind from integer arrays (numpy or torch: xp), as fp32."""
    f32 = xp.float32

    def cast(a):  # exact: every integer here is below 2^24
        return a.astype(f32) if xp is np else a.to(f32)

    uni = cast(m - (1 << 23)) * (2.0 ** -23) * 4.0
    sgn = xp.where((m >> 10) & 1 == 1, -1, 1)
    large = cast(32768 + 32 * (m & 1023))
    subn = cast(sgn * (m & 1023)) * (2.0 ** -24)
    tiny = cast(m & 0xFFFF) * (2.0 ** -40)
    canc = cast((m0 & 0xFFFFF) - (1 << 19)) * (2.0 ** -19) * (1.0 if r % 2 == 0 else -1.0)
    k = m & 63
    inf = float("inf")
    spec = xp.where(k == 0, inf, xp.where(k == 1, -inf, xp.where(k == 2, float("nan"), uni)))
    out = xp.where(cat == 0, large, xp.where(cat == 1, subn, xp.where(cat == 2, tiny, xp.where(
        cat == 3, canc, xp.where(cat == 4, spec, uni)))))
    return out.astype(f32) if xp is np else out.to(f32)


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
        elif kind == "edge":
            u0 = _mix_t((idx + int(_base_np(seed, 0, t))) & M32)
            v = _edge(u0 & 7, m, u0 >> 8, r, torch)
        else:
            v = torch.tensor(scale, dtype=torch.float32, device=out.device) * \
                ((m - (1 << 23)).to(torch.float32) * (2.0 ** -23))
        flat[s0:s1].copy_(v.to(out.dtype))
    return out
