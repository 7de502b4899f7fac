"""N=1 fused pack/x1/N/unpack step on fcn220m (configs[1]) with and without the NEXT-2
statistics epilogue: device ms per step (CUDA events around K steps, gr_wait_async between).

  python tools/bench_local.py [--steps 20] [--stats 0|1|both]"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--stats", default="both")
    ap.add_argument("--buffer", default="f16")
    a = ap.parse_args()
    import torch

    from paper_1909_11150_b200 import GR_F16, GR_F32, Context
    from workloads import fcn220m

    torch.cuda.set_device(0)
    f = fcn220m()
    grads = [torch.randn(int(n), device="cuda") for n in f.numel]
    ptrs = [g.data_ptr() for g in grads]
    res = {}
    for stats in ([0, 1] if a.stats == "both" else [int(a.stats)]):
        ctx = Context(rank=0, world_size=1, device=0, numel=f.numel, group_of=f.group_of,
                      buffer_dtype=GR_F16 if a.buffer == "f16" else GR_F32)
        if stats:
            ctx.gr_enable_grad_stats(True)
        batch = ctx.prepare_batch(list(range(f.T)), ptrs)

        def step():
            ctx.gr_mark_ready_prepared(batch)
            ctx.gr_step(bits=False)
            ctx.gr_wait_async()

        for _ in range(3):
            step()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(a.steps):
            step()
        e1.record()
        torch.cuda.synchronize()
        res[f"ms_per_step_stats{stats}"] = round(e0.elapsed_time(e1) / a.steps, 4)
        ctx.gr_finalize()
    print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
