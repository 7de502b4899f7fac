"""Coordination-cycle latency microbenchmark: host wall time of one gr_step
and the bitvector kernel's own %globaltimer span, at N=1 (a real rank) or N virtual ranks of one
GPU (--virtual N; one host thread per rank).

  python tools/bench_cycle.py [--T 68] [--virtual N] [--iters 2000] [--release]

--release: every cycle marks all T tensors (8 elements each) and releases them (bitvector +
fused data kernel + gr_wait); default: nothing is marked, so the data kernel exits at once and
the cycle is pure coordination (populate, AND, release decision, host hand-off)."""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--T", type=int, default=68)
    ap.add_argument("--G", type=int, default=10)
    ap.add_argument("--virtual", type=int, default=1)
    ap.add_argument("--iters", type=int, default=2000)
    ap.add_argument("--release", action="store_true")
    a = ap.parse_args()
    import torch

    from paper_1909_11150_b200 import GR_F16, Context, virtual_world
    from tests.parity_lib import run_ranks

    torch.cuda.set_device(0)
    T, G, N = a.T, min(a.G, a.T), a.virtual
    group_of = [t * G // T for t in range(T)]
    numel = [8] * T
    if N == 1:
        ctxs = [Context(rank=0, world_size=1, device=0, numel=numel, group_of=group_of, buffer_dtype=GR_F16)]
    else:
        ctxs = virtual_world(world_size=N, device=0, numel=numel, group_of=group_of, buffer_dtype=GR_F16)
    bufs = [torch.zeros(T * 8, device="cuda") for _ in range(N)]
    torch.cuda.synchronize()

    def rank(r):
        c = ctxs[r]
        batch = c.prepare_batch(list(range(T)), [bufs[r].data_ptr() + 32 * t for t in range(T)])
        lat = []
        for i in range(a.iters + 50):
            if a.release:
                c.gr_mark_ready_prepared(batch)
            t0 = time.perf_counter_ns()
            c.gr_step(bits=False)
            t1 = time.perf_counter_ns()
            if a.release:
                c.gr_wait()
            if i == 49:
                c.reset_stats()
            if i >= 50:
                lat.append((t1 - t0) / 1e3)
        if not a.release:
            c.gr_wait()
        st = c.stats()
        return lat, st.bitvector_device_us / max(1, st.cycles), st.host_wait_us / max(1, st.cycles)

    out = run_ranks(N, rank)
    lat = np.concatenate([np.array(o[0]) for o in out])
    res = {"N": N, "virtual": N > 1, "T": T, "G": G, "release": a.release, "iters": a.iters,
           "gr_step_us_p50": round(float(np.percentile(lat, 50)), 2),
           "gr_step_us_p99": round(float(np.percentile(lat, 99)), 2),
           "bitvector_kernel_span_us_mean": round(float(np.mean([o[1] for o in out])), 2),
           "host_wait_us_mean": round(float(np.mean([o[2] for o in out])), 2)}
    print(json.dumps(res), flush=True)
    for c in ctxs:
        c.gr_finalize()


if __name__ == "__main__":
    main()
