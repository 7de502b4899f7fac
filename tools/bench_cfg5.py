"""cfg5 (BASELINE.json configs[4]): grouped-allreduce message-size sweep vs NCCL.

  torchrun --nproc-per-node N tools/bench_cfg5.py [--buffer f16|f32] [--min-kib 1] [--max-mib 1024]

One group holding one contiguous fp32 gradient tensor of S/p_b elements. For every
size: our path (gr_mark_ready -> gr_step -> fused pack/reduce/unpack -> gr_wait;
one-shot and two-shot forced, plus the library's default choice) against torch
NCCL all_reduce(AVG) on an fp16/fp32 tensor of the same message size (reduce only;
no pack/unpack). Device time with CUDA events, max over ranks; busbw = S*2(N-1)/N/t.
Rank 0 prints one JSON line per size and a summary line.
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--buffer", default="f16", choices=["f16", "f32"])
    ap.add_argument("--min-kib", type=int, default=1)
    ap.add_argument("--max-mib", type=int, default=1024)
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--quick", action="store_true", help="library default only, no NCCL (tuning sweeps)")
    ap.add_argument("--tensors", type=int, default=1, help="split the message into this many tensors "
                    "(separate allocations) of one group (SURVEY.md cfg5's 16-tensor variant)")
    a = ap.parse_args()

    import torch
    import torch.distributed as dist

    import paper_1909_11150_b200 as gr

    rank = int(os.environ["RANK"])
    N = int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    pb = 2 if a.buffer == "f16" else 4
    ag = gr.make_allgather(None, local)
    comp = torch.cuda.current_stream(dev)

    def tmax(x):
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def timed(fn, iters):
        for _ in range(3):
            fn()
        dist.barrier(device_ids=[local])
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(comp)
        for _ in range(iters):
            fn()
        e1.record(comp)
        torch.cuda.synchronize()
        return tmax(e0.elapsed_time(e1) / iters)

    sizes = []
    s = a.min_kib * 1024
    while s <= a.max_mib * 1024 * 1024:
        sizes.append(s)
        s *= 2
    rows = []
    for S in sizes:
        n = S // pb
        iters = a.iters if S <= (64 << 20) else max(5, a.iters // 4)
        k = max(1, min(a.tensors, n // 8))
        sizes_t = [n // k + (1 if i < n % k else 0) for i in range(k)]
        gs = [torch.randn(m, device=dev) for m in sizes_t]
        res = {"bytes": S, "elems": n, "tensors": k}
        variants = (("default", -1),) if a.quick else (("default", -1), ("oneshot", 1 << 62), ("twoshot", 0))
        for name, osm in variants:
            ctx = gr.Context(rank=rank, world_size=N, device=local, numel=sizes_t, group_of=[0] * k,
                             buffer_dtype=gr.GR_F16 if pb == 2 else gr.GR_F32, compute_stream=comp.cuda_stream,
                             one_shot_max_bytes=osm, timeout_ms=30000, allgather=ag)
            batch = ctx.prepare_batch(list(range(k)), [x.data_ptr() for x in gs])

            def ours():  # stream-ordered wait: the production contract (host never blocks on the data)
                ctx.gr_mark_ready_prepared(batch)
                ctx.gr_step(bits=False)
                ctx.gr_wait_async()

            def ours_drain():  # every tensor marked: the device-driven cycle, no host round trip
                ctx.gr_mark_ready_prepared(batch)
                ctx.gr_step_drain()
                ctx.gr_wait_async()

            def ours_blocking():
                ctx.gr_mark_ready_prepared(batch)
                ctx.gr_step(bits=False)
                ctx.gr_wait()

            ms = timed(ours, iters)
            res[f"{name}_us"] = ms * 1e3
            res[f"{name}_busbw"] = S * 2 * (N - 1) / N / (ms * 1e-3) / 1e9
            if name == "default":
                res["default_drain_us"] = timed(ours_drain, iters) * 1e3
                res["default_drain_busbw"] = S * 2 * (N - 1) / N / (res["default_drain_us"] * 1e-6) / 1e9
            if name == "default" and not a.quick:
                res["default_blocking_us"] = timed(ours_blocking, iters) * 1e3
            ctx.gr_finalize()
        if not a.quick:
            x = torch.zeros(n, dtype=torch.float16 if pb == 2 else torch.float32, device=dev)
            ms = timed(lambda: dist.all_reduce(x, op=dist.ReduceOp.AVG), iters)
            res["nccl_us"] = ms * 1e3
            res["nccl_busbw"] = S * 2 * (N - 1) / N / (ms * 1e-3) / 1e9
        rows.append(res)
        if rank == 0:
            print(json.dumps({k: (round(v, 3) if isinstance(v, float) else v) for k, v in res.items()}), flush=True)
    if rank == 0:
        print(json.dumps({"cfg5_summary": True, "N": N, "buffer": a.buffer,
                          "what": "ours = mark+gr_step+fused pack/reduce/unpack+gr_wait_async on one fp32 tensor "
                                  "(default_drain_us: gr_step_drain instead of gr_step, no host round trip; "
                                  "default_blocking_us: with the host-blocking gr_wait); "
                                  "nccl = all_reduce(AVG) on a same-size buffer-dtype tensor (reduce only)"}))
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
