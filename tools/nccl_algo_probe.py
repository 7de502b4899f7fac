"""NCCL all_reduce(AVG) busbw at a few sizes under the algorithm NCCL_ALGO selects (run once per
NCCL_ALGO value; NCCL_DEBUG=INFO shows what the default picks). Device time, max over ranks.

  torchrun --nproc-per-node N tools/nccl_algo_probe.py [--sizes-mib 16,64,256] [--dtype f16]
"""
import argparse
import json
import os


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sizes-mib", default="8,16,32,64,128,256")
    ap.add_argument("--dtype", default="f16")
    ap.add_argument("--iters", type=int, default=20)
    a = ap.parse_args()
    import torch
    import torch.distributed as dist
    rank, N = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    dt = torch.float16 if a.dtype == "f16" else torch.float32
    out = {"N": N, "NCCL_ALGO": os.environ.get("NCCL_ALGO", "default"), "dtype": a.dtype}
    for mib in [int(x) for x in a.sizes_mib.split(",")]:
        S = mib << 20
        x = torch.zeros(S // (2 if dt == torch.float16 else 4), dtype=dt, device=dev)
        for _ in range(5):
            dist.all_reduce(x, op=dist.ReduceOp.AVG)
        torch.cuda.synchronize()
        dist.barrier(device_ids=[local])
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(a.iters):
            dist.all_reduce(x, op=dist.ReduceOp.AVG)
        e1.record()
        torch.cuda.synchronize()
        t = torch.tensor([e0.elapsed_time(e1) / a.iters], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
        out[f"{mib}M_us"] = round(ms * 1e3, 1)
        out[f"{mib}M_busbw"] = round(S * 2 * (N - 1) / N / (ms * 1e-3) / 1e9, 1)
    if rank == 0:
        print(json.dumps(out), flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
