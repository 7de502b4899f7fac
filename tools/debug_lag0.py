"""Reproduce a data-kernel stall on virtual ranks and dump the producers' state (GR_DEBUG_DUMP).

  GR_LAG1=0 GR_LAG2=148 GR_DEBUG_DUMP=gpurun_out/dbg python tools/debug_lag0.py [--n 4] [--mib 16]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=4)
    ap.add_argument("--mib", type=int, default=16)
    ap.add_argument("--iters", type=int, default=20)
    a = ap.parse_args()
    import torch

    from paper_1909_11150_b200 import GR_F16, GrError, virtual_world
    from tests.parity_lib import run_ranks
    torch.cuda.set_device(0)
    n = (a.mib << 20) // 2
    ctxs = virtual_world(world_size=a.n, device=0, numel=[n], group_of=[0], buffer_dtype=GR_F16,
                         one_shot_max_bytes=0, timeout_ms=4000)
    gs = [torch.randn(n, device="cuda") for _ in range(a.n)]

    def one(r):
        try:
            for _ in range(a.iters):
                ctxs[r].gr_mark_ready(0, gs[r].data_ptr())
                ctxs[r].gr_step(bits=False)
                ctxs[r].gr_wait()
            return "ok"
        except GrError as e:
            return repr(e)

    print(run_ranks(a.n, one, timeout=120), flush=True)
    for c in ctxs:
        c.gr_finalize()


if __name__ == "__main__":
    main()
