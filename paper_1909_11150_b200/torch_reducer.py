"""PyTorch integration: the paper's gradient path inside a real
autograd backward pass.

`GroupedGradReducer` registers a post-accumulate-grad hook on every parameter; the hook marks
the gradient ready with `gr_mark_ready_async` on the stream autograd is using, so the ready
flag is written by the GPU right after the gradient exists ("pending requests").
`synchronize()` then runs coordination cycles ("tics") as groups become ready —
complete groups are reduced while the GPU is still running the rest of the backward pass — ends
the step with one device-driven drain cycle (`gr_step_drain`), and makes the current stream
wait for the reduced gradients (no host block). One backward pass per `synchronize()`; every
parameter must receive a gradient (a hook that never fires leaves its group unreleased).

Argument marshalling only: all arithmetic runs in libgr.so. Groups default to the paper's
usage — a few contiguous groups of roughly equal bytes in reverse registration order (the
order backward produces gradients; SPEC.md:296 default), or explicit per-parameter group ids
("explicit assignment of collective operations into groups").
"""
from __future__ import annotations

import time

import torch

from .binding import GR_F16, Context, make_allgather


def contiguous_groups(numels, n_groups: int):
    """Group ids for tensors listed in registration order: G contiguous runs of about equal
    element count over the REVERSE order (the order backward produces gradients), numbered in
    that production order (group 0 is ready first)."""
    T = len(numels)
    n_groups = max(1, min(n_groups, T))
    total = float(sum(numels))
    gid = [0] * T
    acc = 0.0
    g = 0
    for i, t in enumerate(reversed(range(T))):
        gid[t] = g
        acc += numels[t]
        remaining_tensors = T - i - 1
        if acc >= (g + 1) * total / n_groups and g < n_groups - 1 and remaining_tensors >= n_groups - 1 - g:
            g += 1
    # make ids dense (a group may have ended up empty on tiny tables)
    remap = {v: k for k, v in enumerate(sorted(set(gid)))}
    return [remap[v] for v in gid]


def drive_cycles(step, drain, wait_group, ready_order, G: int, drain_tail: int = 1, cycle_us: float = 0.0,
                 max_cycles: int = 1_000_000) -> int:
    """The host side of one step's coordination (argument marshalling around gr_step).

    Cycles are driven by local readiness: for each group, in the order its last gradient was
    produced on this rank (`ready_order`), wait_group(g) blocks until it exists, then cycles run
    until g is released (a peer that is behind holds the cycle on the device only for the skew).
    Once at most `drain_tail` groups are left, drain() (gr_step_drain) ends the step without the
    host waiting for the tail of backward. `cycle_us` > 0 polls with fixed-period cycles instead
    (the paper's cycle time).

    Every decision to cycle, stop or drain depends only on the released set, which the global
    AND makes identical on every rank, so all ranks issue the same sequence of collective calls
    whatever their local readiness order (tests/test_torch_reducer.py). Returns the cycles run."""
    n, complete = 0, False
    released = set()

    def cycle():
        nonlocal n, complete
        rel, complete = step()
        n += 1
        released.update(rel)

    if cycle_us > 0:
        nxt = time.perf_counter()
        while n < max_cycles and G - len(released) > drain_tail:
            cycle()
            if complete:
                break
            nxt += cycle_us * 1e-6
            while time.perf_counter() < nxt:
                pass
    else:
        for g in ready_order:
            if complete or G - len(released) <= drain_tail or n >= max_cycles:
                break
            if g in released:
                continue
            wait_group(g)  # the group's gradients exist on this rank
            while g not in released and n < max_cycles:
                cycle()
                if complete or G - len(released) <= drain_tail:
                    break
    if not complete:
        drain()  # every hook has fired: all marks are issued
        n += 1
    return n


class GroupedGradReducer:
    """comm_ctas bounds the SMs a reduction occupies while backward is still running (0 = every
    SM; the fused kernel holds a large shared-memory ring, so each of its CTAs displaces compute
    on its SM); the step's final, device-driven cycle (gr_step_drain) always uses every SM.
    Defaults (4 groups, full grid, per-group cycles, drain of the last group) are the best
    overlapped setting measured on a 51M-parameter FC-DenseNet at N=2/4 (tools/bench_train.py,
    profiles/r01_train/); at that scale one drain cycle after backward
    (`synchronize(drain_tail=n_groups)`) is ~1% faster still."""

    def __init__(self, params, *, rank: int, world_size: int, device: int, groups=None, n_groups: int = 4,
                 buffer_dtype: int = GR_F16, pg=None, timeout_ms: int = 0, comm_ctas: int = 0):
        self.params = [p for p in params if p.requires_grad]
        numels = [p.numel() for p in self.params]
        self.group_of = list(groups) if groups is not None else contiguous_groups(numels, n_groups)
        grad_f16 = [p.dtype == torch.float16 for p in self.params]
        if any(p.dtype not in (torch.float32, torch.float16) for p in self.params):
            raise TypeError("GroupedGradReducer supports fp32 and fp16 parameters")
        self.world_size = world_size
        self._ag = make_allgather(pg, device) if world_size > 1 else None
        self.ctx = Context(rank=rank, world_size=world_size, device=device, numel=numels, group_of=self.group_of,
                           grad_f16=grad_f16, buffer_dtype=buffer_dtype,
                           compute_stream=torch.cuda.current_stream(device).cuda_stream, timeout_ms=timeout_ms,
                           comm_ctas=comm_ctas, allgather=self._ag)
        self.cycles_last_step = 0
        self.G = len(set(self.group_of))
        self._gsize = [0] * self.G
        for g in self.group_of:
            self._gsize[g] += 1
        self._left = list(self._gsize)
        self._ready_order = []  # groups in the order their last gradient was produced (host view)
        self._events = [torch.cuda.Event() for _ in range(self.G)]
        self._hooks = [p.register_post_accumulate_grad_hook(self._make_hook(t)) for t, p in enumerate(self.params)]

    def _make_hook(self, t: int):
        g = self.group_of[t]

        def hook(p):
            # stream-ordered readiness: the flag is written after the accumulation kernel
            stream = torch.cuda.current_stream(p.device)
            self.ctx.gr_mark_ready_async(t, p.grad.data_ptr(), stream.cuda_stream)
            self._left[g] -= 1
            if self._left[g] == 0:  # the group's last gradient: an event tells the host when
                self._events[g].record(stream)
                self._ready_order.append(g)
        return hook

    def synchronize(self, cycle_us: float = 0.0, drain_tail: int = 1, max_cycles: int = 1_000_000):
        """Coordinate the step's reduction while backward is still running on the GPU
        (see drive_cycles), then order the current stream after it. Returns the cycles run."""
        def step():
            rel, complete, _bits, _info = self.ctx.gr_step(bits=False)
            return rel, complete

        n = drive_cycles(step, self.ctx.gr_step_drain, lambda g: self._events[g].synchronize(),
                         self._ready_order, self.G, drain_tail, cycle_us, max_cycles)
        self.ctx.gr_wait_async()
        self._left = list(self._gsize)
        self._ready_order = []
        self.cycles_last_step = n
        return n

    def close(self):
        for h in self._hooks:
            h.remove()
        self._hooks = []
        self.ctx.gr_finalize()
