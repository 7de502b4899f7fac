"""fcn220m: FC-DenseNet-shaped gradient tensor table.

The paper gives three anchors only: an FC-DenseNet with growth k=256, 1024
input channels and avg-pool (§6.2), "22x10^7" weights
 and 1.717x10^13 forward conv ops per step at 512x512
(Table 1). Per-layer sizes are never printed, so this table is a
fit: a Tiramisu-style net with c0=128 and dense blocks (1,4,4,8,4,4,1); each
block layer is a 3x3 conv with K=256, transition-down a 1x1 conv (+avg-pool),
transition-up a 3x3 transposed conv, final a 1x1 conv to one channel.
34 convs, 225,100,032 weights + 15,105 biases = 225,115,137 elements.

Tensor ids follow forward order: tensor 2l is layer l's weight, 2l+1 its bias.
Gradients are released in reverse-layer order (backprop). Groups are the
per-level groups g0..g9 of SURVEY.md Appendix A, numbered in release order.

Synthetic backward delay per layer: d_l = 2*OPS_l / (0.70 * 1401.8e12) s with
OPS_l = 2*H*W*C*K*R*S (Eq.1): backprop-kernel + backprop-input
at 70% of the measured sustained bf16 peak (PAPER.md:196 reports 70% of peak).
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np


@dataclass
class Layer:
    name: str
    C: int
    K: int
    R: int
    H: int
    level: str  # group key

    @property
    def weight_elems(self) -> int:
        return self.C * self.K * self.R * self.R

    @property
    def ops_fwd(self) -> float:
        return 2.0 * self.H * self.H * self.C * self.K * self.R * self.R  # Eq.1


@dataclass
class FcnTable:
    layers: list
    numel: np.ndarray          # [T] int64, tensor id = 2*layer + (0 weight | 1 bias)
    names: list
    group_of: np.ndarray       # [T] int32
    group_names: list
    release_order: list        # layer indices, first released first
    bwd_delay_s: np.ndarray    # [n_layers] synthetic backward time per layer
    extra: dict = field(default_factory=dict)

    @property
    def T(self) -> int:
        return int(self.numel.size)

    @property
    def G(self) -> int:
        return len(self.group_names)


def _layers(k: int = 256, c0: int = 128, cin: int = 1024, hw: int = 512):
    L = []
    L.append(Layer("conv0", cin, c0, 3, hw, "g9"))
    blocks_down = [1, 4, 4]
    c = c0
    h = hw
    skips = []
    tdnames = ["td0", "td1", "td2"]
    dbgroup = ["g9", "g8", "g7"]
    for b, n in enumerate(blocks_down):
        for i in range(n):
            L.append(Layer(f"db{b}.{i}", c + i * k, k, 3, h, dbgroup[b]))
        c = c + n * k
        skips.append((c, h))
        L.append(Layer(tdnames[b], c, c, 1, h, dbgroup[b]))
        h //= 2
    # bottleneck (8 layers) at the lowest resolution
    for i in range(8):
        L.append(Layer(f"bott.{i}", c + i * k, k, 3, h, "g6"))
    new = 8 * k
    blocks_up = [4, 4, 1]
    tugroup = ["g5", "g3", "g1"]
    ubgroup = ["g4", "g2", "g0"]
    for b, n in enumerate(blocks_up):
        skip_c, skip_h = skips[len(skips) - 1 - b]
        L.append(Layer(f"tu{b}", new, new, 3, skip_h, tugroup[b]))
        h = skip_h
        c = new + skip_c
        for i in range(n):
            L.append(Layer(f"ub{b}.{i}", c + i * k, k, 3, h, ubgroup[b]))
        new = n * k
    L.append(Layer("final", new, 1, 1, h, "g0"))
    return L


def fcn220m(sustained_tflops: float = 1401.8, frac_of_peak: float = 0.70) -> FcnTable:
    layers = _layers()
    T = 2 * len(layers)
    numel = np.zeros(T, dtype=np.int64)
    names = []
    for l, ly in enumerate(layers):
        numel[2 * l] = ly.weight_elems
        numel[2 * l + 1] = ly.K
        names += [ly.name + ".w", ly.name + ".b"]
    group_names = [f"g{i}" for i in range(10)]
    group_of = np.array([group_names.index(layers[t // 2].level) for t in range(T)], dtype=np.int32)
    release_order = list(range(len(layers) - 1, -1, -1))
    delay = np.array([2.0 * ly.ops_fwd / (frac_of_peak * sustained_tflops * 1e12) for ly in layers])
    return FcnTable(layers, numel, names, group_of, group_names, release_order, delay,
                    extra={"ops_fwd_total": sum(ly.ops_fwd for ly in layers)})
