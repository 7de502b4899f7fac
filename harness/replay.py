"""Replay a mark schedule through the C ABI on this rank.

mark_cycle[t] = number of gr_step calls this rank completes before it calls
gr_mark_ready(t) (-1: never). The loop ends when step_complete is reported
(identically on every rank) or after max_cycles gr_step calls.
"""
from __future__ import annotations

from dataclasses import dataclass, field


@dataclass
class ReplayLog:
    A: list = field(default_factory=list)         # per cycle: list of W u32 words
    released: list = field(default_factory=list)  # per cycle: ascending group ids
    complete: bool = False
    n_cycles: int = 0


def replay_step(ctx, mark_cycle, ptrs, max_cycles: int = 1000, async_stream=None,
                drain_after: int = -1, before_step=None) -> ReplayLog:
    """drain_after >= 0: after that many gr_step cycles (unless the step completed), mark every
    remaining tensor in schedule order and end the step with one gr_step_drain.
    before_step(): called before every gr_step (e.g. to let stream-ordered marks land, so the
    cycle sees exactly the schedule's marks, as the oracle assumes)."""
    by_cycle: dict[int, list[int]] = {}
    for t, m in enumerate(mark_cycle):
        if m >= 0:
            by_cycle.setdefault(int(m), []).append(t)
    log = ReplayLog()
    c = 0
    while c < max_cycles:
        if c == drain_after:
            for cc in sorted(k for k in by_cycle if k >= c):
                for t in by_cycle[cc]:
                    if async_stream is None:
                        ctx.gr_mark_ready(t, ptrs[t])
                    else:
                        ctx.gr_mark_ready_async(t, ptrs[t], async_stream)
            ctx.gr_step_drain()
            c += 1
            log.complete = True
            break
        for t in by_cycle.get(c, []):
            if async_stream is None:
                ctx.gr_mark_ready(t, ptrs[t])
            else:
                ctx.gr_mark_ready_async(t, ptrs[t], async_stream)
        if before_step is not None:
            before_step()
        rel, complete, A, _info = ctx.gr_step()
        log.A.append(A)
        log.released.append(rel)
        c += 1
        if complete:
            log.complete = True
            break
    log.n_cycles = c
    ctx.gr_wait()
    return log


def make_grads(numel, r: int, seed: int, device, grad_f16=None, kind: str = "uniform"):
    """This rank's seeded gradient tensors (counter-based generator, workloads.values)."""
    import torch

    from workloads.values import fill_values_torch, tensor_scales

    s = tensor_scales(seed, len(numel))
    out = []
    for t, n in enumerate(numel):
        dt = torch.float16 if (grad_f16 is not None and grad_f16[t]) else torch.float32
        x = torch.empty(int(n), dtype=dt, device=device)
        fill_values_torch(x, seed, r, t, float(s[t]), kind)
        out.append(x)
    return out
