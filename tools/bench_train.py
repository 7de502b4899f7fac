"""NEXT-3: scaling efficiency (X1) of a real FC-DenseNet
training step with the grouped bitvector reducer against PyTorch DDP (NCCL buckets).

  torchrun --nproc-per-node N tools/bench_train.py --impl ours|ddp|ddp_fp16|none [--batch 4]

One training step = forward (bf16 autocast) -> MSE loss -> backward -> gradient averaging ->
SGD step, weak scaling (fixed per-GPU batch). `ours`: GroupedGradReducer (post-accumulate
hooks -> gr_mark_ready_async; a cycle as each group's gradients exist on this rank, the last
--drain-tail groups by one device-driven gr_step_drain; fp16 wire);
`ddp`: DistributedDataParallel (fp32 NCCL all_reduce of 25 MB buckets, overlapped with
backward); `ddp_fp16`: the same with the fp16 compression hook (same wire precision as ours);
`none`: no gradient exchange (the N=1 reference for efficiency). Device time with CUDA
events, max over ranks. Prints one JSON line (rank 0).
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--impl", default="ours", choices=["ours", "ddp", "ddp_fp16", "none"])
    ap.add_argument("--batch", type=int, default=4)
    ap.add_argument("--hw", type=int, default=64)
    ap.add_argument("--k", type=int, default=192)
    ap.add_argument("--groups", type=int, default=4)
    ap.add_argument("--cycle-us", type=float, default=0.0, help="0: cycles driven by local group readiness")
    ap.add_argument("--comm-ctas", type=int, default=0)
    ap.add_argument("--drain-tail", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--profile", default="", help="rank 0: torch.profiler chrome trace of 3 steps to this path")
    a = ap.parse_args()

    import torch
    import torch.distributed as dist

    from harness.fcdensenet import make_model

    rank = int(os.environ.get("RANK", "0"))
    N = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if N > 1:
        dist.init_process_group("nccl", device_id=dev)
    torch.backends.cudnn.benchmark = True
    kw = dict(c_in=64, c0=256, k=a.k, blocks=(3, 3, 4, 3, 3))
    model = make_model(7, dev, **kw)
    n_params = sum(p.numel() for p in model.parameters())
    g = torch.Generator(device="cpu").manual_seed(1000 + rank)
    x = torch.randn(a.batch, kw["c_in"], a.hw, a.hw, generator=g).to(dev)
    y = torch.randn(a.batch, 1, a.hw, a.hw, generator=g).to(dev)

    red = None
    net = model
    if a.impl == "ours" and N > 1:
        from paper_1909_11150_b200.torch_reducer import GroupedGradReducer
        red = GroupedGradReducer(model.parameters(), rank=rank, world_size=N, device=local, n_groups=a.groups,
                                 comm_ctas=a.comm_ctas)
    elif a.impl in ("ddp", "ddp_fp16") and N > 1:
        net = torch.nn.parallel.DistributedDataParallel(model, device_ids=[local], gradient_as_bucket_view=True)
        if a.impl == "ddp_fp16":
            from torch.distributed.algorithms.ddp_comm_hooks import default_hooks
            net.register_comm_hook(None, default_hooks.fp16_compress_hook)
    opt = torch.optim.SGD(model.parameters(), lr=1e-3)
    comp = torch.cuda.current_stream(dev)

    def step():
        opt.zero_grad(set_to_none=False)
        with torch.autocast("cuda", dtype=torch.bfloat16):
            out = net(x)
        loss = torch.nn.functional.mse_loss(out.float(), y)
        loss.backward()
        if red is not None:
            red.synchronize(cycle_us=a.cycle_us, drain_tail=a.drain_tail)
        opt.step()

    def tmax(v):
        if N == 1:
            return v
        t = torch.tensor([v], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    for _ in range(a.warmup):
        step()
    torch.cuda.synchronize()
    if N > 1:
        dist.barrier(device_ids=[local])
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(comp)
    cycles = 0
    for _ in range(a.steps):
        step()
        cycles += red.cycles_last_step if red is not None else 0
    e1.record(comp)
    torch.cuda.synchronize()
    ms = tmax(e0.elapsed_time(e1) / a.steps)
    if rank == 0:
        print(json.dumps({"bench": "train_fcdensenet", "impl": a.impl, "n_gpus": N, "batch_per_gpu": a.batch,
                          "hw": a.hw, "k": a.k, "params": n_params, "grad_mb_fp32": round(n_params * 4 / 2**20, 1),
                          "tensors": len(list(model.parameters())), "groups": a.groups if red else None,
                          "cycle_us": a.cycle_us if red else None, "comm_ctas": a.comm_ctas if red else None,
                          "drain_tail": a.drain_tail if red else None, "ms_per_step": round(ms, 3),
                          "samples_per_s": round(N * a.batch / (ms * 1e-3), 1),
                          "cycles_per_step": cycles / a.steps if red else None}), flush=True)
    if a.profile:
        from torch.profiler import ProfilerActivity, profile
        with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
            for _ in range(3):
                step()
            torch.cuda.synchronize()
        if rank == 0:
            prof.export_chrome_trace(a.profile)
    if red is not None:
        red.close()
    if N > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
