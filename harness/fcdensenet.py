"""A small FC-DenseNet (Tiramisu-style encoder-decoder with dense blocks, §6.2)
used as a real gradient producer for the autograd integration tests (NEXT-3). Same topology
family as the fcn220m table (workloads/fcn.py) at toy width: dense blocks of 3x3 convs with
growth k, 1x1 transition-down + avg-pool, 3x3 transposed-conv transition-up, skip concat,
1x1 output conv. Deterministic init from a seed."""
from __future__ import annotations

import torch
import torch.nn as nn


class DenseBlock(nn.Module):
    def __init__(self, c_in: int, k: int, n: int):
        super().__init__()
        self.layers = nn.ModuleList([nn.Conv2d(c_in + i * k, k, 3, padding=1) for i in range(n)])

    def forward(self, x):
        new = []
        for conv in self.layers:
            y = torch.relu(conv(x))
            new.append(y)
            x = torch.cat([x, y], 1)
        return x, torch.cat(new, 1)


class TinyFCDenseNet(nn.Module):
    def __init__(self, c_in: int = 8, c0: int = 16, k: int = 8, blocks=(2, 2, 3, 2, 2)):
        super().__init__()
        down, bott, up = blocks[:2], blocks[2], blocks[3:]
        self.conv0 = nn.Conv2d(c_in, c0, 3, padding=1)
        self.down_blocks = nn.ModuleList()
        self.tds = nn.ModuleList()
        c = c0
        skips = []
        for n in down:
            self.down_blocks.append(DenseBlock(c, k, n))
            c = c + n * k
            skips.append(c)
            self.tds.append(nn.Conv2d(c, c, 1))
        self.bott = DenseBlock(c, k, bott)
        new = bott * k
        self.tus = nn.ModuleList()
        self.up_blocks = nn.ModuleList()
        for i, n in enumerate(up):
            self.tus.append(nn.ConvTranspose2d(new, new, 3, stride=2, padding=1, output_padding=1))
            c = new + skips[len(skips) - 1 - i]
            self.up_blocks.append(DenseBlock(c, k, n))
            new = n * k
        self.final = nn.Conv2d(new, 1, 1)

    def forward(self, x):
        x = self.conv0(x)
        skips = []
        for blk, td in zip(self.down_blocks, self.tds):
            x, _ = blk(x)
            skips.append(x)
            x = nn.functional.avg_pool2d(td(x), 2)
        _, x = self.bott(x)
        for tu, blk in zip(self.tus, self.up_blocks):
            x = torch.cat([tu(x), skips.pop()], 1)
            _, x = blk(x)
        return self.final(x)


def make_model(seed: int, device, **kw) -> TinyFCDenseNet:
    torch.manual_seed(seed)
    return TinyFCDenseNet(**kw).to(device)


def batch(seed: int, rank: int, device, n: int = 2, c_in: int = 8, hw: int = 32):
    g = torch.Generator(device="cpu").manual_seed(seed * 1000003 + rank)
    x = torch.randn(n, c_in, hw, hw, generator=g)
    y = torch.randn(n, 1, hw, hw, generator=g)
    return x.to(device), y.to(device)
