"""The N-rank data path on ONE GPU (virtual ranks, gr_init_virtual): fcn220m through the fused
pack -> reduce -> x1/N -> unpack kernel (xfer_kernel_v), timed with CUDA events; every "peer"
read is a local HBM read, so the kernel is HBM-bound and its efficiency is the HBM efficiency of
the pack / reduce-scatter / all-gather-unpack stages that a real N>1 run overlaps with NVLink
(those stages' HBM efficiency had never been measured).

  python tools/bench_virtual.py [--n 2] [--algo twoshot|oneshot] [--steps 10] [--push]

Algorithmic HBM bytes per launch (all ranks), E elements per rank, p_g = 4, p_b = 2 (fp16 wire):
  two-shot, per rank: PACK (N-1)/N*E*(p_g+p_b) + RS E/N*((N-1)*p_b + 2*p_g + p_b)
                      + AG (N-1)/N*E*(p_b+p_g)
  one-shot, per rank: PACK E*(p_g+p_b) + RED E*((N-1)*p_b + 2*p_g)
(push: the same bytes, the packed copies written into the receivers' slots instead of read).
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
    ap.add_argument("--n", type=int, default=2)
    ap.add_argument("--algo", default="twoshot", choices=["twoshot", "oneshot"])
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    a = ap.parse_args()
    import numpy as np
    import torch

    from paper_1909_11150_b200 import GR_F16, virtual_world
    from tests.parity_lib import run_ranks
    from workloads import fcn220m
    from workloads.values import fill_values_torch, tensor_scales

    torch.cuda.set_device(0)
    dev = torch.device("cuda", 0)
    f = fcn220m()
    N = a.n
    E = int(f.numel.sum())
    s = tensor_scales(1, f.T)
    grads = []
    for r in range(N):
        gr_ = []
        for t in range(f.T):
            x = torch.empty(int(f.numel[t]), dtype=torch.float32, device=dev)
            fill_values_torch(x, 1, r, t, float(s[t]))
            gr_.append(x)
        grads.append(gr_)
    torch.cuda.synchronize()
    osm = 0 if a.algo == "twoshot" else (1 << 62)
    ctxs = virtual_world(world_size=N, device=0, numel=f.numel, group_of=f.group_of, buffer_dtype=GR_F16,
                         one_shot_max_bytes=osm, timeout_ms=60000)
    order = [t for l in f.release_order for t in (2 * l, 2 * l + 1)]
    batches = [c.prepare_batch(order, [grads[r][t].data_ptr() for t in order]) for r, c in enumerate(ctxs)]

    def step(r):
        c = ctxs[r]
        c.gr_mark_ready_prepared(batches[r])
        rel, complete, _A, _ = c.gr_step(bits=False)
        assert complete
        c.gr_wait()

    for _ in range(a.warmup):
        run_ranks(N, step)
    for c in ctxs:
        c.set_timing(True)
        c.reset_stats()
    t0 = time.perf_counter()
    for _ in range(a.steps):
        run_ranks(N, step)
    wall = (time.perf_counter() - t0) / a.steps
    # each rank brackets the one combined launch with events on its own stream; the last rank to
    # arrive brackets it most tightly (the others also count the wait for that rank)
    kern_ms = min(c.stats().data_kernel_ms / max(1, c.stats().data_launches) for c in ctxs)
    pg, pb = 4, 2
    if a.algo == "twoshot":
        per_rank = (N - 1) / N * E * (pg + pb) + E / N * ((N - 1) * pb + 2 * pg + pb) + (N - 1) / N * E * (pb + pg)
    else:
        per_rank = E * (pg + pb) + E * ((N - 1) * pb + 2 * pg)
    alg = per_rank * N
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    gbs = alg / (kern_ms * 1e-3) / 1e9
    print(json.dumps({"virtual_ranks": N, "algo": a.algo, "push": os.environ.get("GR_PUSH", "0"),
                      "workload": "fcn220m x N ranks on one GPU", "elements_per_rank": E,
                      "kernel_ms": round(kern_ms, 4), "wall_ms_per_step": round(wall * 1e3, 3),
                      "algorithmic_hbm_bytes_per_launch": int(alg), "achieved_GBps": round(gbs, 1),
                      "peak_GBps": peaks["hbm_gbs"], "frac": round(gbs / peaks["hbm_gbs"], 4)}), flush=True)
    for c in ctxs:
        c.gr_finalize()


if __name__ == "__main__":
    main()
