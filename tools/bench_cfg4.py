"""cfg4 (BASELINE.json configs[3]): bitvector-only cycle latency, T = 64 .. 65,536.

  torchrun --nproc-per-node N tools/bench_cfg4.py [--cycles 10000] [--skew-us 0,10,100]

T = 2^6 .. 2^16 (11 points) tensors of 8 elements, G = T/8 contiguous groups of 8; rank r marks in reverse order
rotated by r*T/N ("adversarial skew": a group completes only when the slowest rank's
rotation reaches it), T/16 marks per cycle. The last rank is a straggler that enters
gr_step delta us late every cycle. Reported per T: host latency of gr_step (p50/p99; for
the straggler this is last arrival -> its result), the bitvector kernel's own span
(%globaltimer), and the same-box baselines: NCCL all_reduce(MIN) on u8[T] ready flags
(NCCL has no bitwise AND), gloo all_reduce(BAND) on u32[W] (the paper's MPI_BAND), and the
paper's original master-worker coordination (harness/master_worker.py: Gatherv of serialized
requests to rank 0, intersect, Bcast of ordered responses; gloo on the host CPU).
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def pct(xs, q):
    xs = sorted(xs)
    return xs[min(len(xs) - 1, int(q * len(xs)))]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cycles", type=int, default=10000)
    ap.add_argument("--baseline-cycles", type=int, default=10000)
    ap.add_argument("--tstep", type=int, default=2, help="T multiplier between points (2: all 11)")
    ap.add_argument("--skew-us", default="0,10,100")
    ap.add_argument("--tmax", type=int, default=65536)
    ap.add_argument("--tmin", type=int, default=64)
    ap.add_argument("--no-baselines", action="store_true")
    a = ap.parse_args()

    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_1909_11150_b200 as gr
    from harness.master_worker import MasterWorker
    from workloads import cfg4_case

    rank = int(os.environ["RANK"])
    N = int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    gloo = dist.new_group(backend="gloo")
    ag = gr.make_allgather(None, local)
    straggler = N - 1

    def spin(us):
        t = time.perf_counter() + us * 1e-6
        while time.perf_counter() < t:
            pass

    T = a.tmin
    while T <= a.tmax:
        case = cfg4_case(T, N)
        grads = torch.zeros(T * 8, device=dev)
        ptrs = [grads.data_ptr() + 32 * t for t in range(T)]
        ctx = gr.Context(rank=rank, world_size=N, device=local, numel=[8] * T, group_of=case.group_of,
                         buffer_dtype=gr.GR_F16, timeout_ms=30000, allgather=ag)
        order = {}
        for t in range(T):
            order.setdefault(int(case.mark_cycle[rank, t]), []).append(t)
        for skew in [float(x) for x in a.skew_us.split(",")]:
            lat, kern = [], []
            done = 0
            dist.barrier(device_ids=[local])
            while done < a.cycles:
                c = 0
                while True:
                    ids = order.get(c, [])
                    if ids:
                        ctx.gr_mark_ready_batch(ids, [ptrs[t] for t in ids])
                    if rank == straggler and skew > 0:
                        spin(skew)
                    s0 = ctx.stats().bitvector_device_us
                    t0 = time.perf_counter()
                    _rel, complete, _A, _ = ctx.gr_step(bits=False)
                    lat.append((time.perf_counter() - t0) * 1e6)
                    kern.append(ctx.stats().bitvector_device_us - s0)
                    c += 1
                    done += 1
                    if complete:
                        break
                ctx.gr_wait()
            res = {"T": T, "W": ctx.W, "G": T // 8, "N": N, "skew_us": skew, "cycles": len(lat),
                   "gr_step_us_p50": pct(lat, 0.5), "gr_step_us_p99": pct(lat, 0.99),
                   "kernel_us_p50": pct(kern, 0.5), "kernel_us_p99": pct(kern, 0.99)}
            allres = [None] * N
            dist.all_gather_object(allres, res)
            if rank == 0:
                st = allres[straggler]
                out = {"T": T, "N": N, "skew_us": skew, "W": res["W"],
                       "straggler_gr_step_us_p50": round(st["gr_step_us_p50"], 2),
                       "straggler_gr_step_us_p99": round(st["gr_step_us_p99"], 2),
                       "rank0_gr_step_us_p50": round(allres[0]["gr_step_us_p50"], 2),
                       "kernel_us_p50": round(max(r["kernel_us_p50"] for r in allres), 2),
                       "kernel_us_p99": round(max(r["kernel_us_p99"] for r in allres), 2)}
                print(json.dumps(out), flush=True)
        ctx.gr_finalize()
        if a.no_baselines:
            T *= a.tstep
            continue
        # baselines on the same box
        flags = torch.ones(T, dtype=torch.uint8, device=dev)
        for _ in range(20):
            dist.all_reduce(flags, op=dist.ReduceOp.MIN)
        torch.cuda.synchronize()
        nl = []
        nb = max(300, a.baseline_cycles)
        for _ in range(nb):
            t0 = time.perf_counter()
            dist.all_reduce(flags, op=dist.ReduceOp.MIN)
            flags.cpu()  # the host needs the result, as gr_step's caller does
            nl.append((time.perf_counter() - t0) * 1e6)
        words = torch.ones((T + 2 + 31) // 32, dtype=torch.int32)
        gl = []
        for i in range(nb):
            t0 = time.perf_counter()
            dist.all_reduce(words, op=dist.ReduceOp.BAND, group=gloo)
            gl.append((time.perf_counter() - t0) * 1e6)
        # the paper's original strategy (NEXT-4): master-worker gather -> intersect -> broadcast
        # of serialized requests/responses over gloo, same schedule, every cycle timed
        mw = MasterWorker(rank, N, case.group_of, pg=gloo)
        ml, mcyc = [], 0
        dist.barrier(group=gloo)
        while mcyc < a.baseline_cycles:
            c = 0
            while True:
                t0 = time.perf_counter()
                _ids, complete = mw.cycle(order.get(c, []))
                ml.append((time.perf_counter() - t0) * 1e6)
                c += 1
                mcyc += 1
                if complete:
                    break
        mw_p = torch.tensor([pct(ml, 0.5), pct(ml, 0.99)], dtype=torch.float64)
        dist.all_reduce(mw_p, op=dist.ReduceOp.MAX, group=gloo)
        if rank == 0:
            print(json.dumps({"T": T, "N": N, "baseline": True,
                              "nccl_min_u8_us_p50": round(pct(nl[50:], 0.5), 2),
                              "nccl_min_u8_us_p99": round(pct(nl[50:], 0.99), 2),
                              "gloo_band_u32_us_p50": round(pct(gl[50:], 0.5), 2),
                              "gloo_band_u32_us_p99": round(pct(gl[50:], 0.99), 2),
                              "baseline_cycles": nb,
                              "master_worker_us_p50": round(float(mw_p[0]), 2),
                              "master_worker_us_p99": round(float(mw_p[1]), 2),
                              "master_worker_cycles": len(ml)}), flush=True)
        T *= a.tstep
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
