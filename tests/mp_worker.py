"""torchrun worker for the multi-GPU parity tests (one process per GPU).

  torchrun --nproc-per-node N --master-addr 127.0.0.1 tests/mp_worker.py --suite cfg1 --seeds 0:20

Every rank replays the same seeded schedules through the C ABI, checks its own
schedule and values against the oracle (tests/parity_lib.py) and the ranks
compare output hashes (bitwise-identical replicas). Exit code 0 = all passed.
"""
from __future__ import annotations

import argparse
import os
import sys
import traceback

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def autograd_suite(rank, N, local, dev):
    """NEXT-3: the reducer driven by real backward hooks of a small FC-DenseNet. Reduced
    gradients match the fp64 average of every rank's plain-backward gradient within the fp16
    tolerance; replicas stay bitwise identical through SGD steps; the loss goes down."""
    import hashlib

    import numpy as np
    import torch
    import torch.distributed as dist

    from harness.fcdensenet import batch, make_model
    from paper_1909_11150_b200.torch_reducer import GroupedGradReducer

    ok = True
    torch.backends.cudnn.deterministic = True
    torch.backends.cudnn.benchmark = False
    model = make_model(3, dev)
    ref = make_model(3, dev)
    red = GroupedGradReducer(model.parameters(), rank=rank, world_size=N, device=local, n_groups=4)
    opt = torch.optim.SGD(model.parameters(), lr=0.05)
    losses = []
    for step in range(4):
        x, y = batch(step, rank, dev)
        opt.zero_grad(set_to_none=False)
        loss = torch.nn.functional.mse_loss(model(x), y)
        loss.backward()
        cycles = red.synchronize()
        torch.cuda.synchronize()
        # reference: plain backward on an identical replica, then the exact fp64 average
        ref.load_state_dict(model.state_dict()) if step == 0 else None
        ref.zero_grad(set_to_none=False)
        torch.nn.functional.mse_loss(ref(x), y).backward()
        for p_ours, p_ref in zip(model.parameters(), ref.parameters()):
            mine = p_ref.grad.detach().double().cpu().contiguous()
            g_all = [torch.empty_like(mine) for _ in range(N)]
            dist.all_gather(g_all, mine)  # gloo process group: CPU tensors
            stack = torch.stack(g_all)
            want = stack.mean(0)
            # north-star fp16 bound plus the fp16 subnormal quantum: real gradients of this toy
            # model reach |g| ~ 1e-6, where RN to fp16 has absolute error up to 2^-25 per rounding
            # (input + output rounding -> 2^-24); R11
            tol = 2.0 ** -10 * N * float(stack.abs().max()) + 2.0 ** -24
            err = float((p_ours.grad.double().cpu() - want).abs().max())
            if err > tol:
                ok = False
                print(f"[rank {rank}] step {step}: reduced gradient off by {err} > {tol}", flush=True)
        opt.step()
        ref.load_state_dict(model.state_dict())
        red_loss = torch.tensor([loss.item()], dtype=torch.float64)
        dist.all_reduce(red_loss)
        losses.append(float(red_loss) / N)
        h = hashlib.sha256(b"".join(p.detach().cpu().numpy().tobytes() for p in model.parameters())).hexdigest()
        hs = [None] * N
        dist.all_gather_object(hs, h)
        if len(set(hs)) != 1:
            ok = False
            print(f"[rank {rank}] step {step}: replicas diverged", flush=True)
    if rank == 0:
        print(f"autograd suite: losses {losses}, cycles last step {cycles}", flush=True)
    red.close()
    return ok


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--suite", default="cfg1")
    ap.add_argument("--seeds", default="0:10")
    ap.add_argument("--buffers", default="f16,f32")
    ap.add_argument("--one-shot-max-bytes", type=int, default=-1)
    ap.add_argument("--chunk-elems", type=int, default=0)
    args = ap.parse_args()

    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_1909_11150_b200 import GR_F16, GR_F32, Context, make_allgather
    from tests.parity_lib import check_grad_stats, run_case_on_rank
    from workloads import cfg1_case, fcn220m
    from workloads.schedules import Case, random_mark_schedule, random_partition, reverse_layer_schedule

    rank = int(os.environ["RANK"])
    N = int(os.environ["WORLD_SIZE"])
    # one process per GPU: never time-share a device between spinning ranks (Xid 109 risk on
    # this pool); the N-rank path on fewer GPUs is tests/test_gpu_virtual.py's job
    local = int(os.environ.get("LOCAL_RANK", rank))
    if local >= torch.cuda.device_count():
        raise SystemExit(f"rank {rank}: LOCAL_RANK {local} but only {torch.cuda.device_count()} GPUs")
    torch.cuda.set_device(local)
    dist.init_process_group("gloo")
    ag = make_allgather(None)
    dev = torch.device("cuda", local)
    s0, s1 = (int(x) for x in args.seeds.split(":"))
    failures = 0
    ncase = 0

    def run(case, seed, buf, grad_f16=None, kind="uniform", chunk=0, osm=None, max_cycles=None, stats=False):
        nonlocal failures, ncase
        ncase += 1
        ctx = Context(rank=rank, world_size=N, device=local, numel=case.numel, group_of=case.group_of,
                      grad_f16=grad_f16, buffer_dtype=GR_F16 if buf == "f16" else GR_F32,
                      one_shot_max_bytes=args.one_shot_max_bytes if osm is None else osm,
                      chunk_elems=chunk or args.chunk_elems, timeout_ms=20000, allgather=ag)
        if stats:
            ctx.gr_enable_grad_stats(True)
        ok = True
        nvls, why = ctx.nvls()
        if os.environ.get("GR_NVLS") == "1" and not nvls:
            raise RuntimeError(f"GR_NVLS=1 but NVLS is not enabled: {why}")
        try:
            _log, h = run_case_on_rank(ctx, case, rank, seed, dev, buf == "f16", grad_f16, kind,
                                       max_cycles=max_cycles, exact=not nvls)
            if stats:
                ss = check_grad_stats(ctx, case, seed, buf == "f16", grad_f16, kind, exact=not nvls,
                                      where=f"rank {rank} seed {seed}")
                all_ss = [None] * N
                dist.all_gather_object(all_ss, ss)
                for other in all_ss:  # fp64 atomics: equal up to summation order (~1e-15)
                    for a, b in zip(ss, other):
                        assert abs(a - b) <= 1e-12 * max(abs(a), abs(b)) + 1e-300, \
                            f"rank {rank} seed {seed}: statistics differ across ranks {a!r} {b!r}"
        except AssertionError as e:
            ok = False
            h = "FAIL"
            print(f"[rank {rank}] seed {seed} buf {buf}: {e}", flush=True)
        hs = [None] * N
        dist.all_gather_object(hs, h)
        if ok and len(set(hs)) != 1:
            ok = False
            print(f"[rank {rank}] seed {seed} buf {buf}: outputs differ across ranks {hs}", flush=True)
        failures += (not ok)
        ctx.gr_finalize()

    try:
        for buf in args.buffers.split(","):
            if args.suite == "cfg1":
                for seed in range(s0, s1):
                    case = cfg1_case(seed, N=N)
                    run(case, seed, buf)
            elif args.suite == "edge":
                # ragged sizes, many chunks, both algorithms, fp16 grads, integer payloads
                for seed in range(s0, s1):
                    rng = np.random.default_rng(seed)
                    T = int(rng.integers(1, 24))
                    G = int(rng.integers(1, T + 1))
                    numel = rng.integers(1, 200000, size=T).astype(np.int64)
                    numel[rng.integers(0, T)] = int(rng.integers(1, 9))
                    case = Case(N, numel, random_partition(T, G, rng), random_mark_schedule(N, T, seed, 3), seed)
                    gf = (rng.random(T) < 0.3).tolist()
                    for osm in (0, 1 << 62):  # force two-shot, force one-shot
                        run(case, seed, buf, grad_f16=gf, chunk=int(rng.choice([1024, 4096, 32768])), osm=osm)
                    run(case, seed, buf, kind="int", osm=0)
            elif args.suite == "stats":
                for seed in range(s0, s1):
                    rng = np.random.default_rng(seed + 77)
                    T = int(rng.integers(2, 20))
                    numel = rng.integers(1, 300000, size=T).astype(np.int64)
                    case = Case(N, numel, random_partition(T, int(rng.integers(1, T + 1)), rng),
                                random_mark_schedule(N, T, seed, 3), seed)
                    gf = (rng.random(T) < 0.3).tolist()
                    for osm in (0, 1 << 62):
                        run(case, seed, buf, grad_f16=gf, osm=osm, stats=True)
            elif args.suite == "bigT":  # bitvectors beyond the inline size, up to T = 65,536
                from workloads import cfg4_case
                for seed in range(s0, s1):
                    for T, rand_groups in ((4096, True), (65536, False)):
                        base = cfg4_case(T, N, marks_per_cycle=T // 5)
                        rng = np.random.default_rng(T + seed)
                        group_of = random_partition(T, T // 8, rng) if rand_groups else base.group_of
                        numel = rng.integers(1, 64, size=T).astype(np.int64)
                        run(Case(N, numel, group_of, base.mark_cycle, seed), seed, buf)
            elif args.suite == "drain":
                from tests.parity_lib import run_drain_case_on_rank
                stream = torch.cuda.Stream(device=dev)
                for seed in range(s0, s1):
                    case = cfg1_case(seed, N=N)
                    ncase += 1
                    ctx = Context(rank=rank, world_size=N, device=local, numel=case.numel, group_of=case.group_of,
                                  buffer_dtype=GR_F16 if buf == "f16" else GR_F32, timeout_ms=20000, allgather=ag)
                    ok = True
                    try:
                        _log, h = run_drain_case_on_rank(ctx, case, rank, seed, dev, buf == "f16", seed % 3,
                                                         async_stream=stream.cuda_stream if seed % 2 else None)
                    except AssertionError as e:
                        ok, h = False, "FAIL"
                        print(f"[rank {rank}] drain seed {seed} buf {buf}: {e}", flush=True)
                    hs = [None] * N
                    dist.all_gather_object(hs, h)
                    if ok and len(set(hs)) != 1:
                        ok = False
                        print(f"[rank {rank}] drain seed {seed}: outputs differ across ranks", flush=True)
                    failures += (not ok)
                    ctx.gr_finalize()
            elif args.suite == "autograd":
                ncase += 1
                ok = autograd_suite(rank, N, local, dev)
                failures += (not ok)
            elif args.suite == "fcn":
                f = fcn220m()
                mark = reverse_layer_schedule(len(f.layers), N, f.release_order, layers_per_cycle=1,
                                              jitter_seed=s0, max_shift=2)
                case = Case(N, f.numel, f.group_of, mark, s0)
                run(case, s0, buf)              # library default (one-shot below the crossover)
                if buf == "f16" and os.environ.get("GR_NVLS") != "1":
                    run(case, s0, buf, osm=0)   # every group through the two-shot path
            else:
                raise SystemExit(f"unknown suite {args.suite}")
    except Exception:
        traceback.print_exc()
        failures += 1
    tot = [None] * N
    dist.all_gather_object(tot, failures)
    if rank == 0:
        print(f"mp_worker suite={args.suite} N={N} cases={ncase} failures={sum(tot)} "
              f"GR_NVLS={os.environ.get('GR_NVLS', 'default')}", flush=True)
    dist.destroy_process_group()
    sys.exit(1 if sum(tot) else 0)


if __name__ == "__main__":
    main()
