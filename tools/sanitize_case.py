"""Small cases of every kernel of the path, for compute-sanitizer (one tool per gpurun call).

  compute-sanitizer --tool memcheck|racecheck|synccheck|initcheck python tools/sanitize_case.py [--quick]

N=1: cfg1-shaped steps through gr_mark_ready / gr_step / gr_wait (bitvector_kernel,
local_kernel, fp16 and fp32 buffers, statistics epilogue on) and one stream-ordered drain
cycle. Virtual ranks on the one GPU (gr_init_virtual: bitvector_kernel_v, xfer_kernel_v):
N=2 two-shot and one-shot, N=4 two-shot with ragged tensors spanning several chunks (the TMA
ring, the slow piece path, the publisher ring). Every case is still checked against the
oracle (tests/parity_lib.py), so the run also proves the sanitized kernels computed the right
values. Exits 0 when everything passed.
"""
import argparse
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--quick", action="store_true", help="fewer cases (racecheck is slow)")
    a = ap.parse_args()
    import numpy as np
    import torch

    import paper_1909_11150_b200 as gr
    from tests.parity_lib import run_case_on_rank, run_drain_case_on_rank, run_virtual_case
    from workloads import cfg1_case
    from workloads.schedules import Case, random_mark_schedule

    torch.cuda.set_device(0)
    dev = torch.device("cuda", 0)
    t0 = time.time()
    seeds = (0,) if a.quick else (0, 1)
    for seed in seeds:
        for buf16 in (True, False):
            c = cfg1_case(seed)
            case = Case(1, c.numel, c.group_of, c.mark_cycle[:1].copy(), seed)
            ctx = gr.Context(rank=0, world_size=1, device=0, numel=case.numel, group_of=case.group_of,
                             buffer_dtype=gr.GR_F16 if buf16 else gr.GR_F32, timeout_ms=120000)
            ctx.gr_enable_grad_stats(True)
            run_case_on_rank(ctx, case, 0, seed, dev, buf16)
            ctx.gr_finalize()
            print(f"N=1 cfg1 seed {seed} buf16={buf16} ok ({time.time() - t0:.0f} s)", flush=True)
    # drain cycle with stream-ordered marks
    c = cfg1_case(5)
    case = Case(1, c.numel, c.group_of, c.mark_cycle[:1].copy(), 5)
    ctx = gr.Context(rank=0, world_size=1, device=0, numel=case.numel, group_of=case.group_of,
                     buffer_dtype=gr.GR_F16, timeout_ms=120000)
    s = torch.cuda.Stream(dev)
    run_drain_case_on_rank(ctx, case, 0, 5, dev, True, 1, async_stream=s.cuda_stream)
    ctx.gr_finalize()
    print(f"N=1 drain ok ({time.time() - t0:.0f} s)", flush=True)

    for seed, osm in ((3, 0), (4, 1 << 62)):
        run_virtual_case(cfg1_case(seed, N=2), seed, dev, True, one_shot_max_bytes=osm, timeout_ms=120000,
                         stats=True)
        print(f"virtual N=2 {'two' if osm == 0 else 'one'}-shot ok ({time.time() - t0:.0f} s)", flush=True)
    if not a.quick:
        rng = np.random.default_rng(7)
        T, N = 6, 4
        numel = rng.integers(1, 70000, T).astype(np.int64)
        group_of = np.array([0, 0, 1, 1, 1, 2], dtype=np.int32)
        mark = random_mark_schedule(N, T, 7, 3)
        case = Case(N, numel, group_of, mark, 7)
        run_virtual_case(case, 7, dev, True, one_shot_max_bytes=0, timeout_ms=120000, chunk_elems=8192)
        print(f"virtual N=4 two-shot ragged ok ({time.time() - t0:.0f} s)", flush=True)
    torch.cuda.synchronize()
    print("sanitize cases ok", flush=True)


if __name__ == "__main__":
    main()
