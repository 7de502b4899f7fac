"""GPU parity: the CUDA path (through the C ABI) against the oracle.

N=1 cases run in-process on cuda:0. N>1 cases launch tests/mp_worker.py
under torchrun (one process per GPU) and are skipped when the box has fewer
GPUs; the same N-rank path is covered on one GPU by tests/test_gpu_virtual.py
(virtual ranks, one launch over all ranks). Both paths check schedule bit-exactness, value bit-exactness against the
oracle's emulation, the north-star tolerances and cross-rank identity
(tests/parity_lib.py).
"""
import os
import subprocess
import sys

import numpy as np
import pytest

from tests.conftest import ROOT, gpu_count
from workloads import cfg1_case, fcn220m
from workloads.schedules import Case, random_mark_schedule, random_partition, reverse_layer_schedule

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def gpu():
    if gpu_count() < 1:
        pytest.skip("no GPU")
    import torch
    torch.cuda.set_device(0)
    return torch.device("cuda", 0)


def _ctx(case, buf16, **kw):
    from paper_1909_11150_b200 import GR_F16, GR_F32, Context
    return Context(rank=0, world_size=1, device=0, numel=case.numel, group_of=case.group_of,
                   buffer_dtype=GR_F16 if buf16 else GR_F32, timeout_ms=5000, **kw)


def _n1(case):
    return Case(1, case.numel, case.group_of, case.mark_cycle[:1].copy(), case.seed)


@pytest.mark.parametrize("buf16", [True, False])
def test_cfg1_n1_many_seeds(gpu, buf16):
    from tests.parity_lib import run_case_on_rank
    for seed in range(40):
        case = _n1(cfg1_case(seed))
        ctx = _ctx(case, buf16)
        run_case_on_rank(ctx, case, 0, seed, gpu, buf16)
        ctx.gr_finalize()


def test_same_context_many_steps(gpu):
    """Epoch handling: the same context across 6 steps with different schedules."""
    from tests.parity_lib import run_case_on_rank
    base = cfg1_case(3)
    ctx = _ctx(_n1(base), True)
    for step in range(6):
        mark = random_mark_schedule(1, base.T, 100 + step)
        case = Case(1, base.numel, base.group_of, mark, 100 + step)
        run_case_on_rank(ctx, case, 0, 100 + step, gpu, True)
    assert ctx.stats().steps == 6
    ctx.gr_finalize()


@pytest.mark.parametrize("seed", range(6))
def test_edge_shapes_n1(gpu, seed):
    """Ragged sizes (1..7 elements, non-multiples of 8), tensors spanning many
    chunks, tiny chunks, fp16 gradients, integer payloads, G=1 and singletons."""
    from tests.parity_lib import run_case_on_rank
    rng = np.random.default_rng(seed)
    T = int(rng.integers(1, 30))
    numel = rng.integers(1, 300000, size=T).astype(np.int64)
    numel[: min(T, 3)] = rng.integers(1, 8, size=min(T, 3))
    G = [1, T, int(rng.integers(1, T + 1))][seed % 3]
    case = Case(1, numel, random_partition(T, G, rng), random_mark_schedule(1, T, seed, 3), seed)
    gf = (rng.random(T) < 0.4).tolist()
    for buf16 in (True, False):
        for chunk in (8, 1024, 32768):
            ctx = _ctx(case, buf16, chunk_elems=chunk, grad_f16=gf)
            run_case_on_rank(ctx, case, 0, seed, gpu, buf16, grad_f16=gf)
            ctx.gr_finalize()
        ctx = _ctx(case, buf16)
        run_case_on_rank(ctx, case, 0, seed, gpu, buf16, kind="int")
        ctx.gr_finalize()


def test_unaligned_pointer_scalar_path(gpu):
    """A gradient view starting 1 element into its storage takes the scalar path."""
    import torch
    from paper_1909_11150_b200 import GR_F16, Context
    from tests.parity_lib import check_values
    n = 10001
    base = torch.empty(n + 1, device=gpu)
    base.uniform_(-1, 1)
    g = base[1:]
    src = g.cpu().numpy().copy()
    ctx = Context(rank=0, world_size=1, device=0, numel=[n], group_of=[0], buffer_dtype=GR_F16)
    ctx.gr_mark_ready(0, g.data_ptr())
    rel, complete, A, _ = ctx.gr_step()
    ctx.gr_wait()
    assert rel == [0] and complete and A == [0b111]
    check_values(g.cpu().numpy(), [src], 1, True, False)
    ctx.gr_finalize()


def test_never_marked_and_errors(gpu):
    import torch
    from paper_1909_11150_b200 import GR_F16, Context, GrError
    from paper_1909_11150_b200.binding import GR_EINVAL, GR_ESTATE, GR_EABORT
    x = torch.zeros(64, device=gpu)
    ctx = Context(rank=0, world_size=1, device=0, numel=[64, 64], group_of=[0, 1], buffer_dtype=GR_F16)
    ctx.gr_mark_ready(0, x.data_ptr())
    with pytest.raises(GrError) as e:
        ctx.gr_mark_ready(0, x.data_ptr())          # duplicate mark
    assert e.value.code == GR_ESTATE
    with pytest.raises(GrError) as e:
        ctx.gr_mark_ready(5, x.data_ptr())          # bad id
    assert e.value.code == GR_EINVAL
    with pytest.raises(GrError) as e:
        ctx.gr_mark_ready(1, x.data_ptr(), rank=1)  # wrong rank
    assert e.value.code == GR_EINVAL
    for _ in range(3):                              # tensor 1 never marked: group 1 stays pending
        rel, complete, A, _ = ctx.gr_step()
        assert not complete
    ctx.gr_set_status(abort=True)
    with pytest.raises(GrError) as e:
        ctx.gr_step()
    assert e.value.code == GR_EABORT
    with pytest.raises(GrError) as e:               # sticky
        ctx.gr_step()
    assert e.value.code == GR_ESTATE
    ctx.gr_finalize()


def test_async_wait_pipelined_steps(gpu):
    """gr_wait_async: 5 back-to-back steps without host blocking; the reduction is idempotent
    at N=1 (re-rounding), so the final values equal one oracle application."""
    import torch
    from tests.parity_lib import check_values, host_inputs
    from harness.replay import make_grads
    case = _n1(cfg1_case(11))
    ctx = _ctx(case, True)
    grads = make_grads(case.numel, 0, 11, gpu)
    order = list(range(case.T))
    for _ in range(5):
        ctx.gr_mark_ready_batch(order, [g.data_ptr() for g in grads])
        rel, complete, _, _ = ctx.gr_step()
        assert complete and rel == list(range(case.G))
        ctx.gr_wait_async()
    torch.cuda.synchronize()
    for t in range(case.T):
        check_values(grads[t].cpu().numpy(), host_inputs(case.numel, 1, 11, t, False), 1, True, False)
    assert ctx.stats().steps == 5
    ctx.gr_finalize()


@pytest.mark.parametrize("buf16", [True, False])
def test_grad_stats_epilogue_n1(gpu, buf16):
    """NEXT-2: fused ||g||^2 per tensor and non-finite flag, checked against the oracle."""
    import math
    from tests.parity_lib import check_grad_stats, run_case_on_rank
    from harness.replay import make_grads
    rng = np.random.default_rng(5)
    T = 12
    numel = rng.integers(1, 200000, size=T).astype(np.int64)
    case = Case(1, numel, random_partition(T, 4, rng), random_mark_schedule(1, T, 5, 2), 5)
    gf = (rng.random(T) < 0.3).tolist()
    ctx = _ctx(case, buf16, grad_f16=gf)
    ctx.gr_enable_grad_stats(True)
    run_case_on_rank(ctx, case, 0, 5, gpu, buf16, grad_f16=gf)
    check_grad_stats(ctx, case, 5, buf16, grad_f16=gf)
    # a step with an Inf in tensor 3: flag set, that tensor's norm is Inf, the others finite
    grads = make_grads(case.numel, 0, 5, gpu, gf)
    grads[3].view(-1)[min(7, grads[3].numel() - 1)] = float("inf")
    ctx.gr_mark_ready_batch(list(range(T)), [g.data_ptr() for g in grads])
    while True:
        _rel, complete, _, _ = ctx.gr_step()
        if complete:
            break
    ctx.gr_wait()
    sumsq, nonfinite = ctx.gr_grad_stats()
    assert nonfinite and math.isinf(sumsq[3]) and all(math.isfinite(v) for i, v in enumerate(sumsq) if i != 3)
    ctx.gr_finalize()


def test_async_marks_follow_stream(gpu):
    """gr_mark_ready_async: the flag lands only after the stream's prior work."""
    import torch
    from paper_1909_11150_b200 import GR_F32, Context, gr_bench_spin
    s = torch.cuda.Stream(device=gpu)
    x = torch.ones(1024, device=gpu)
    ctx = Context(rank=0, world_size=1, device=0, numel=[1024], group_of=[0], buffer_dtype=GR_F32)
    with torch.cuda.stream(s):
        gr_bench_spin(200_000_000, 4, s.cuda_stream)          # 200 ms of "backward"
        x.mul_(3.0)
    ctx.gr_mark_ready_async(0, x.data_ptr(), s.cuda_stream)
    rel, complete, _, _ = ctx.gr_step()                     # the spin is still running
    assert rel == [] and not complete
    s.synchronize()
    rel, complete, _, _ = ctx.gr_step()
    assert rel == [0] and complete
    ctx.gr_wait()
    assert torch.equal(x, torch.full_like(x, 3.0))
    ctx.gr_finalize()


def test_released_wait_async_orders_copy_out(gpu):
    """gr_released_wait_async: a side stream that waits on it sees each released group's
    reduced values while later groups are still pending (fp16 buffer at N=1: fl32(fl16(g)))."""
    import torch
    from paper_1909_11150_b200 import GR_F16, Context
    n = 1 << 22
    xs = [torch.randn(n, device=gpu) * (i + 1) for i in range(3)]
    want = [x.half().float() for x in xs]
    ctx = Context(rank=0, world_size=1, device=0, numel=[n] * 3, group_of=[0, 1, 2], buffer_dtype=GR_F16)
    side = torch.cuda.Stream(device=gpu)
    outs = [torch.empty_like(x) for x in xs]
    for g in range(3):
        ctx.gr_mark_ready(g, xs[g].data_ptr())
        rel, complete, _, _ = ctx.gr_step()
        assert rel == [g] and complete == (g == 2)
        ctx.gr_released_wait_async(side.cuda_stream)
        with torch.cuda.stream(side):
            outs[g].copy_(xs[g])
    side.synchronize()
    for g in range(3):
        assert torch.equal(outs[g], want[g]), g
    ctx.gr_wait()
    ctx.gr_finalize()


@pytest.mark.parametrize("buf16", [True, False])
def test_step_drain_n1(gpu, buf16):
    """gr_step_drain: the cycles before it follow the oracle's schedule, the drain cycle releases
    every remaining group; values bit-exact. With stream-ordered marks queued behind 50 ms of
    device work the call returns at once and the device waits for the marks."""
    import torch
    from paper_1909_11150_b200 import gr_bench_spin
    from tests.parity_lib import run_drain_case_on_rank
    for seed in range(12):
        case = _n1(cfg1_case(seed))
        ctx = _ctx(case, buf16)
        run_drain_case_on_rank(ctx, case, 0, seed, gpu, buf16, drain_after=seed % 3)
        ctx.gr_finalize()
    case = _n1(cfg1_case(99))
    ctx = _ctx(case, buf16)
    s = torch.cuda.Stream(device=gpu)
    gr_bench_spin(50_000_000, 4, s.cuda_stream)
    run_drain_case_on_rank(ctx, case, 0, 99, gpu, buf16, drain_after=0, async_stream=s.cuda_stream)
    ctx.gr_finalize()


def test_step_drain_requires_every_mark(gpu):
    import torch
    from paper_1909_11150_b200 import GR_F16, Context, GrError
    from paper_1909_11150_b200.binding import GR_ESTATE
    x = torch.zeros(64, device=gpu)
    ctx = Context(rank=0, world_size=1, device=0, numel=[64, 64], group_of=[0, 1], buffer_dtype=GR_F16)
    ctx.gr_mark_ready(0, x.data_ptr())
    with pytest.raises(GrError) as e:
        ctx.gr_step_drain()
    assert e.value.code == GR_ESTATE
    ctx.gr_mark_ready(1, x.data_ptr())
    ctx.gr_step_drain()
    ctx.gr_wait()
    ctx.gr_finalize()


@pytest.mark.parametrize("T,rand_groups", [(4096, True), (65536, False)])
def test_large_tables_n1(gpu, T, rand_groups):
    """Bitvectors beyond the inline-parameter size (W > 64 words: mark bits DMA'd, 1024-thread
    bitvector kernel, thread-per-word populate) up to cfg4's largest table (T = 65,536, W = 2,049):
    schedule and A words bit-exact, values bit-exact; host marks and stream-ordered marks (the
    warp-ballot populate over 65,536 per-tensor flags)."""
    import torch
    from tests.parity_lib import run_case_on_rank
    from workloads import cfg4_case
    base = cfg4_case(T, 1, marks_per_cycle=T // 5)
    rng = np.random.default_rng(T)
    group_of = random_partition(T, T // 8, rng) if rand_groups else base.group_of
    numel = rng.integers(1, 64, size=T).astype(np.int64)
    case = Case(1, numel, group_of, base.mark_cycle, 17)
    for buf16, async_marks in ((True, False), (False, True)):
        ctx = _ctx(case, buf16)
        s = torch.cuda.Stream(device=gpu) if async_marks else None
        # stream-ordered marks become visible when their stream runs the write; letting the
        # stream drain before each cycle makes the cycle see exactly the schedule's marks
        run_case_on_rank(ctx, case, 0, 17, gpu, buf16, async_stream=s.cuda_stream if s else None,
                         before_step=s.synchronize if s else None)
        ctx.gr_finalize()


def test_fcn220m_n1_full_size(gpu):
    """The bench workload at full size (225,115,137 elements, 68 tensors,
    10 groups), reverse-layer schedule; values checked on sampled elements."""
    from tests.parity_lib import run_case_on_rank
    f = fcn220m()
    mark = reverse_layer_schedule(len(f.layers), 1, f.release_order, layers_per_cycle=3)
    case = Case(1, f.numel, f.group_of, mark, 21)
    for buf16 in (True, False):
        ctx = _ctx(case, buf16)
        run_case_on_rank(ctx, case, 0, 21, gpu, buf16)
        ctx.gr_finalize()


def _torchrun(n, *args, timeout=900, env_extra=None):
    env = dict(os.environ, PYTHONPATH=ROOT, **(env_extra or {}))
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(29500 + n), os.path.join(ROOT, "tests", "mp_worker.py"),
           *args]
    r = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=timeout, cwd=ROOT)
    print(r.stdout[-4000:], r.stderr[-4000:])
    return r.returncode


@pytest.mark.parametrize("n", [2, 4, 8])
def test_multi_gpu_cfg1(n):
    if gpu_count() < n:
        pytest.skip(f"needs {n} GPUs")
    assert _torchrun(n, "--suite", "cfg1", "--seeds", "0:30") == 0


@pytest.mark.parametrize("n", [2, 4])
def test_multi_gpu_armed(n):
    """Armed cycles at N>1 (gr.h gr_step): every gap qualifies, so one resident bitvector kernel
    per rank serves cycle after cycle and each data kernel waits for its cycle's record; then
    with the host stalled after each doorbell (the kernel runs ahead and expires unseen)."""
    if gpu_count() < n:
        pytest.skip(f"needs {n} GPUs")
    on = {"GR_ARM": "1", "GR_ARM_GAP_US": "1000000000", "GR_ARM_US": "1000000"}
    assert _torchrun(n, "--suite", "cfg1", "--seeds", "40:50", env_extra=on) == 0
    late = dict(on, GR_ARM_US="100", GR_ARM_RING_DELAY_US="300")
    assert _torchrun(n, "--suite", "cfg1", "--seeds", "50:54", env_extra=late) == 0


@pytest.mark.parametrize("n", [2, 4, 8])
def test_multi_gpu_edge(n):
    if gpu_count() < n:
        pytest.skip(f"needs {n} GPUs")
    assert _torchrun(n, "--suite", "edge", "--seeds", "0:4") == 0
    # the push two-shot variant (off by default) stays parity-green
    assert _torchrun(n, "--suite", "edge", "--seeds", "4:6", env_extra={"GR_PUSH": "1"}) == 0


@pytest.mark.parametrize("n", [2, 4, 8])
def test_multi_gpu_fcn220m(n):
    if gpu_count() < n:
        pytest.skip(f"needs {n} GPUs")
    assert _torchrun(n, "--suite", "fcn", "--seeds", "5:6") == 0


@pytest.mark.parametrize("n", [2, 4, 8])
def test_multi_gpu_nvls(n):
    """NVLS (in-switch reduction) forced on: edge shapes and the full fcn220m set; values
    within the north-star tolerance (the switch's accumulation order is its own), integer
    payloads bit-exact, replicas bitwise identical."""
    if gpu_count() < n:
        pytest.skip(f"needs {n} GPUs")
    assert _torchrun(n, "--suite", "edge", "--seeds", "0:3", env_extra={"GR_NVLS": "1"}) == 0
    assert _torchrun(n, "--suite", "fcn", "--seeds", "7:8", env_extra={"GR_NVLS": "1"}) == 0


@pytest.mark.parametrize("n", [2, 4, 8])
def test_multi_gpu_step_drain(n):
    """gr_step_drain across ranks: host and stream-ordered marks, drain after 0-2 cycles."""
    if gpu_count() < n:
        pytest.skip(f"needs {n} GPUs")
    assert _torchrun(n, "--suite", "drain", "--seeds", "0:12") == 0


@pytest.mark.parametrize("n", [2, 4, 8])
def test_multi_gpu_large_tables(n):
    """W > 64 bitvectors across ranks (T = 4,096 random groups, T = 65,536 cfg4 groups of 8 with
    rank-rotated orders): A words, released lists and values bit-exact, replicas identical."""
    if gpu_count() < n:
        pytest.skip(f"needs {n} GPUs")
    assert _torchrun(n, "--suite", "bigT", "--seeds", "0:1", "--buffers", "f16") == 0


@pytest.mark.parametrize("n", [2, 4, 8])
def test_multi_gpu_grad_stats(n):
    """NEXT-2 epilogue at N ranks: every rank's per-tensor ||g||^2 matches the oracle and the
    other ranks' (every rank holds the full reduced gradient)."""
    if gpu_count() < n:
        pytest.skip(f"needs {n} GPUs")
    assert _torchrun(n, "--suite", "stats", "--seeds", "0:3") == 0


@pytest.mark.parametrize("set_to_none", [False, True])
def test_autograd_reducer_n1(gpu, set_to_none):
    """NEXT-3 at N=1: hooks mark the gradients during backward; after synchronize() each
    gradient equals fl32(fl16(plain-backward gradient)) bit for bit (reading R7-R9 at N=1).
    set_to_none=True is PyTorch's default zero_grad(): every step hands each parameter a NEW
    gradient buffer, so the reducer must reduce the pointers of that step."""
    import torch
    from harness.fcdensenet import batch, make_model
    from paper_1909_11150_b200.torch_reducer import GroupedGradReducer
    torch.backends.cudnn.deterministic = True  # the reference backward must reproduce the gradients
    torch.backends.cudnn.benchmark = False
    model, ref = make_model(3, gpu), make_model(3, gpu)
    red = GroupedGradReducer(model.parameters(), rank=0, world_size=1, device=0, n_groups=3)
    for step in range(3):
        x, y = batch(step, 0, gpu)
        model.zero_grad(set_to_none=set_to_none)
        ref.load_state_dict(model.state_dict())
        ref.zero_grad(set_to_none=False)
        torch.nn.functional.mse_loss(model(x), y).backward()
        red.synchronize()
        torch.nn.functional.mse_loss(ref(x), y).backward()
        torch.cuda.synchronize()
        for a, b in zip(model.parameters(), ref.parameters()):
            assert torch.equal(a.grad, b.grad.half().float())
        with torch.no_grad():
            for p in model.parameters():
                p -= 0.05 * p.grad
    red.close()


@pytest.mark.parametrize("n", [2, 4, 8])
def test_multi_gpu_autograd_reducer(n):
    """NEXT-3 at N ranks: backward hooks + cycles on a small FC-DenseNet; reduced gradients vs
    the fp64 average of the plain-backward gradients, replicas identical through SGD steps."""
    if gpu_count() < n:
        pytest.skip(f"needs {n} GPUs")
    assert _torchrun(n, "--suite", "autograd", "--seeds", "0:1", "--buffers", "f16") == 0


def test_new_gradient_buffers_every_step_async_wait(gpu):
    """Gradient pointers that change every step (PyTorch's default zero_grad(set_to_none=True)
    hands each parameter a new buffer), with gr_wait_async between steps and each step's
    reduction held back behind 20 ms of compute: every step must reduce its OWN buffers. The
    pointer table a cycle uses is snapshotted when the cycle is enqueued (a queued copy from the
    live table would read the next step's pointers). fp16 buffer at N=1: out = fl32(fl16(g))."""
    import torch
    from paper_1909_11150_b200 import GR_F16, Context, gr_bench_spin
    n = 1 << 16
    ctx = Context(rank=0, world_size=1, device=0, numel=[n] * 3, group_of=[0, 1, 2], buffer_dtype=GR_F16)
    kept = []
    for step in range(6):
        gr_bench_spin(20_000_000, 8, 0)               # backward still running on the compute stream
        xs = [torch.randn(n, device=gpu) * (step + 1) for _ in range(3)]
        want = [x.half().float() for x in xs]
        for t in range(3):
            ctx.gr_mark_ready(t, xs[t].data_ptr())
        rel, complete, _, _ = ctx.gr_step()
        assert rel == [0, 1, 2] and complete
        ctx.gr_wait_async()
        kept.append((xs, want))
    torch.cuda.synchronize()
    for step, (xs, want) in enumerate(kept):
        for t in range(3):
            assert torch.equal(xs[t], want[t]), (step, t)
    ctx.gr_finalize()


@pytest.mark.parametrize("arm", ["on", "expire", "off", "late"])
def test_armed_cycles_n1(gpu, arm, monkeypatch):
    """Armed cycles (gr.h gr_step): in a tight cycle loop the next cycle's bitvector kernel is
    launched ahead of the cycle and polls a pinned doorbell; gr_wait / gr_step_drain / timing
    retire it, and an armed kernel that expires before its doorbell hands the cycle back to a
    normal launch. Many-cycle cfg1 schedules (host marks, drains with host or stream-ordered
    marks, a blocking gr_wait per step, timing mode toggled) stay bit-exact against the oracle
    with the armed path always taken ("on": every gap qualifies, the kernel lives 1 s), always
    expiring ("expire": 1 us lifetime), off, and "late": a 100 us lifetime with the host stalled
    300 us after every doorbell, so the resident kernel runs the cycle and expires on the next
    one before the host reads its acknowledgement (the ack word is already one cycle ahead)."""
    import torch
    from paper_1909_11150_b200 import GR_F16, Context
    from tests.parity_lib import run_case_on_rank, run_drain_case_on_rank
    monkeypatch.setenv("GR_ARM", "0" if arm == "off" else "1")
    monkeypatch.setenv("GR_ARM_GAP_US", "1000000000")
    monkeypatch.setenv("GR_ARM_US", {"expire": "1", "late": "100"}.get(arm, "1000000"))
    if arm == "late":
        monkeypatch.setenv("GR_ARM_RING_DELAY_US", "300")
    base = cfg1_case(11)
    ctx = Context(rank=0, world_size=1, device=0, numel=base.numel, group_of=base.group_of, buffer_dtype=GR_F16,
                  timeout_ms=10000)
    s = torch.cuda.Stream(device=gpu)
    try:
        for seed in range(8):
            c = cfg1_case(100 + seed)
            case = Case(1, base.numel, base.group_of, c.mark_cycle[:1].copy(), 100 + seed)
            ctx.set_timing(seed == 3)
            if seed % 4 == 2:
                run_drain_case_on_rank(ctx, case, 0, 100 + seed, gpu, True, 1,
                                       async_stream=s.cuda_stream if seed % 2 else None)
            else:
                run_case_on_rank(ctx, case, 0, 100 + seed, gpu, True)
        st = ctx.stats()
        if arm == "on":
            assert 0 < st.armed_cycles < st.cycles and st.armed_expired == 0
        elif arm == "expire":  # a 1 us lifetime: most armed kernels expire, a few are rung in time
            assert st.armed_expired > 0 and st.armed_cycles + st.armed_expired < st.cycles
        elif arm == "late":  # each armed kernel that is rung runs that cycle, then expires unseen
            assert st.armed_cycles > 0
        else:
            assert st.armed_cycles == 0 and st.armed_expired == 0
    finally:
        ctx.gr_finalize()


@pytest.mark.parametrize("T", [64, 4096])
def test_marks_racing_steps(gpu, T):
    """gr_mark_ready / gr_mark_ready_async from another thread race gr_step (gr.h: thread-safe):
    every cycle takes one consistent snapshot of marks, pointers and the compute fence, so each
    tensor is reduced exactly once with its own pointer. Host marks for even tensors,
    stream-ordered marks for odd ones; random order and timing; fp16 buffer at N=1."""
    import random
    import threading
    import time
    import torch
    from paper_1909_11150_b200 import GR_F16, Context
    rng = np.random.default_rng(T)
    group_of = random_partition(T, max(1, T // 8), rng)
    numel = rng.integers(1, 3000, size=T).astype(np.int64)
    ctx = Context(rank=0, world_size=1, device=0, numel=numel, group_of=group_of, buffer_dtype=GR_F16)
    side = torch.cuda.Stream(device=gpu)
    for step in range(4):
        xs = [torch.randn(int(k), device=gpu) for k in numel]
        want = [x.half().float() for x in xs]
        torch.cuda.synchronize()
        order = list(range(T))
        random.Random(step).shuffle(order)

        def marker():
            r = random.Random(1000 + step)
            for i, t in enumerate(order):
                if t % 2:
                    ctx.gr_mark_ready_async(t, xs[t].data_ptr(), side.cuda_stream)
                else:
                    ctx.gr_mark_ready(t, xs[t].data_ptr())
                if r.random() < 0.05:
                    time.sleep(r.random() * 2e-4)

        th = threading.Thread(target=marker)
        th.start()
        seen = set()
        for _ in range(200000):
            rel, complete, _, _ = ctx.gr_step(bits=False)
            assert not (set(rel) & seen)
            seen |= set(rel)
            if complete:
                break
        th.join()
        assert complete and len(seen) == int(max(group_of)) + 1
        ctx.gr_wait()
        for t in range(T):
            assert torch.equal(xs[t], want[t]), (step, t)
    ctx.gr_finalize()


@pytest.mark.parametrize("buf16", [True, False])
def test_numeric_edges_n1(gpu, buf16):
    """Numeric edge cases element by element against the oracle (workloads.values kind "edge"):
    values near fp16's maximum, fp16 subnormals, values below fp16's smallest subnormal (flushed
    by the pack), +-Inf and NaN (propagated), fp32 and fp16 gradients; bit-exact (NaN payloads
    aside) and within the north-star tolerance on the finite elements."""
    from tests.parity_lib import run_case_on_rank
    rng = np.random.default_rng(41)
    T = 9
    numel = rng.integers(1, 100000, size=T).astype(np.int64)
    case = Case(1, numel, random_partition(T, 3, rng), random_mark_schedule(1, T, 41, 2), 41)
    for gf in (None, [t % 2 == 0 for t in range(T)]):
        ctx = _ctx(case, buf16, grad_f16=gf)
        run_case_on_rank(ctx, case, 0, 41, gpu, buf16, grad_f16=gf, kind="edge")
        ctx.gr_finalize()
