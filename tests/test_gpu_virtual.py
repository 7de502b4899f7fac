"""GPU parity of the N-rank path on ONE GPU: virtual ranks (gr_init_virtual).

N contexts of one process on one B200, one host thread per rank; each cycle's bitvector
kernel and fused pack -> sum-allreduce -> x1/N -> unpack kernel (xfer_kernel: one-shot and
two-shot) run as one launch over all ranks, so every cross-rank step of the method — the AND
of the ranks' bitvectors, the release of complete groups, the
fusion-buffer pack, the rank-order sum and x1/N, the all-gather unpack — runs
on the device at N = 2, 4 and 8 and is checked against the oracle exactly as a process of a
real N-GPU run is (tests/parity_lib.py): A_c and the released lists bit-exact, every reduced
element bit-exact against oracle.emulate and within the north-star tolerance, replicas bitwise
identical. Also the failure paths that need several ranks: a rank that stops stepping
(GR_ETIMEOUT), ABORT / SHUTDOWN raised by one rank (OR over ranks).
"""
import numpy as np
import pytest

from tests.conftest import gpu_count
from workloads import cfg1_case, fcn220m
from workloads.schedules import Case, random_mark_schedule, random_partition, reverse_layer_schedule

pytestmark = pytest.mark.gpu

ONE_SHOT, TWO_SHOT = 1 << 62, 0  # one_shot_max_bytes forcing each algorithm
NS = [2, 3, 4, 8]


@pytest.fixture(scope="module")
def gpu():
    if gpu_count() < 1:
        pytest.skip("no GPU")
    import torch
    torch.cuda.set_device(0)
    return torch.device("cuda", 0)


def _algos(out):
    return {o[4] for o in out}


@pytest.mark.parametrize("n", NS)
@pytest.mark.parametrize("buf16", [True, False])
def test_virtual_cfg1(gpu, n, buf16):
    """configs[0]'s shape (T=8, <=4K elements, G=3, random per-rank orders) at N virtual ranks."""
    from tests.parity_lib import run_virtual_case
    from paper_1909_11150_b200 import GR_ALGO_ONESHOT
    for seed in range(12 if n < 8 else 6):
        out = run_virtual_case(cfg1_case(seed, N=n), seed, gpu, buf16, timeout_ms=20000)
        assert _algos(out) <= {GR_ALGO_ONESHOT}  # small messages take the one-shot path


@pytest.mark.parametrize("n", NS)
def test_virtual_edge_both_algorithms(gpu, n):
    """Ragged sizes, tensors spanning many chunks, fp16 gradients, integer payloads; two-shot
    (owner reduce-scatter + all-gather unpack) and one-shot each forced."""
    from paper_1909_11150_b200 import GR_ALGO_ONESHOT, GR_ALGO_TWOSHOT
    from tests.parity_lib import run_virtual_case
    for seed in range(3):
        rng = np.random.default_rng(seed)
        T = int(rng.integers(1, 24))
        G = int(rng.integers(1, T + 1))
        numel = rng.integers(1, 200000, size=T).astype(np.int64)
        numel[rng.integers(0, T)] = int(rng.integers(1, 9))
        case = Case(n, numel, random_partition(T, G, rng), random_mark_schedule(n, T, seed, 3), seed)
        gf = (rng.random(T) < 0.3).tolist()
        for buf16 in (True, False):
            chunk = int(rng.choice([1024, 4096, 32768]))
            out = run_virtual_case(case, seed, gpu, buf16, grad_f16=gf, chunk_elems=chunk,
                                   one_shot_max_bytes=TWO_SHOT)
            assert _algos(out) == {GR_ALGO_TWOSHOT}
            out = run_virtual_case(case, seed, gpu, buf16, grad_f16=gf, chunk_elems=chunk,
                                   one_shot_max_bytes=ONE_SHOT)
            assert _algos(out) == {GR_ALGO_ONESHOT}
        run_virtual_case(case, seed, gpu, True, kind="int", one_shot_max_bytes=TWO_SHOT)


@pytest.mark.parametrize("n", [2, 3, 4])
def test_virtual_numeric_edges(gpu, n):
    """Numeric edge cases across ranks (kind "edge"): N-rank sums above fp16's range whose mean
    is inside it (reading R8: x1/N before the fp16 store), fp16 subnormal inputs and outputs,
    exact cancellation between ranks (+0), +-Inf / NaN propagation; both algorithms, both
    buffer precisions, fp16 and fp32 gradients — bit-exact against oracle.emulate."""
    from tests.parity_lib import run_virtual_case
    rng = np.random.default_rng(50 + n)
    T = 7
    numel = rng.integers(1, 120000, size=T).astype(np.int64)
    case = Case(n, numel, random_partition(T, 3, rng), random_mark_schedule(n, T, 50 + n, 2), 50 + n)
    gf = [t % 3 == 0 for t in range(T)]
    for buf16 in (True, False):
        for osm in (TWO_SHOT, ONE_SHOT):
            run_virtual_case(case, 50 + n, gpu, buf16, grad_f16=gf, kind="edge", one_shot_max_bytes=osm,
                             chunk_elems=4096)


@pytest.mark.parametrize("n", NS)
def test_virtual_fcn220m_full_size(gpu, n):
    """The bench workload (225,115,137 elements, 68 tensors, 10 groups) at full size, per-rank
    jittered reverse-layer release; the library default algorithm and two-shot forced; values
    on sampled elements (every sampled element recomputed on the host by the oracle)."""
    from tests.parity_lib import run_virtual_case
    f = fcn220m()
    mark = reverse_layer_schedule(len(f.layers), n, f.release_order, layers_per_cycle=1, jitter_seed=n, max_shift=2)
    case = Case(n, f.numel, f.group_of, mark, 30 + n)
    run_virtual_case(case, 30 + n, gpu, True)
    run_virtual_case(case, 30 + n, gpu, True, one_shot_max_bytes=TWO_SHOT)
    if n == 2:
        run_virtual_case(case, 30 + n, gpu, False, one_shot_max_bytes=TWO_SHOT)


@pytest.mark.parametrize("n", NS)
def test_virtual_step_drain(gpu, n):
    """gr_step_drain across virtual ranks after 0-2 host cycles, host and stream-ordered marks."""
    import torch
    from tests.parity_lib import run_virtual_case
    streams = [torch.cuda.Stream(device=gpu).cuda_stream for _ in range(n)]
    for seed in range(6):
        run_virtual_case(cfg1_case(seed, N=n), seed, gpu, seed % 2 == 0, drain_after=seed % 3,
                         async_streams=streams if seed % 2 else None)


@pytest.mark.parametrize("n", [2, 4])
def test_virtual_large_tables(gpu, n):
    """W > 64 bitvectors across ranks (DMA'd mark snapshots, 1024-thread bitvector kernel):
    T = 4,096 random groups and T = 65,536 cfg4 groups of 8 with rank-rotated orders."""
    from tests.parity_lib import run_virtual_case
    from workloads import cfg4_case
    for T, rand_groups in ((4096, True), (65536, False)):
        base = cfg4_case(T, n, marks_per_cycle=T // 5)
        rng = np.random.default_rng(T + n)
        group_of = random_partition(T, T // 8, rng) if rand_groups else base.group_of
        numel = rng.integers(1, 64, size=T).astype(np.int64)
        run_virtual_case(Case(n, numel, group_of, base.mark_cycle, 3), 3, gpu, True)


@pytest.mark.parametrize("n", [2, 4])
def test_virtual_grad_stats(gpu, n):
    """NEXT-2 epilogue at N ranks, both algorithms: every rank's per-tensor ||g||^2 matches the
    oracle and the other ranks'."""
    from tests.parity_lib import run_virtual_case
    for seed in range(2):
        rng = np.random.default_rng(seed + 77)
        T = int(rng.integers(2, 20))
        numel = rng.integers(1, 300000, size=T).astype(np.int64)
        case = Case(n, numel, random_partition(T, int(rng.integers(1, T + 1)), rng),
                    random_mark_schedule(n, T, seed, 3), seed)
        gf = (rng.random(T) < 0.3).tolist()
        for osm in (TWO_SHOT, ONE_SHOT):
            run_virtual_case(case, seed, gpu, True, grad_f16=gf, stats=True, one_shot_max_bytes=osm)


@pytest.mark.parametrize("n", [2, 4])
def test_virtual_many_steps_same_contexts(gpu, n):
    """Epochs and step parity (double-buffered fusion buffers and flag pads) across 5 steps of
    the same virtual world, two-shot, different schedules per step."""
    from paper_1909_11150_b200 import GR_F16, virtual_world
    from tests.parity_lib import run_case_on_rank, run_ranks
    base = cfg1_case(7, N=n)
    ctxs = virtual_world(world_size=n, device=0, numel=base.numel, group_of=base.group_of, buffer_dtype=GR_F16,
                         one_shot_max_bytes=TWO_SHOT, chunk_elems=256)
    try:
        for step in range(5):
            case = Case(n, base.numel, base.group_of, random_mark_schedule(n, base.T, 200 + step, 3), 200 + step)
            hs = run_ranks(n, lambda r: run_case_on_rank(ctxs[r], case, r, 200 + step, gpu, True)[1])
            assert len(set(hs)) == 1
        assert all(c.stats().steps == 5 for c in ctxs)
    finally:
        for c in ctxs:
            c.gr_finalize()


# ------------------------------------------------------------------ push data path (GR_PUSH=1)

@pytest.fixture
def push_mode(monkeypatch):
    """Contexts created inside the test use the push data path: packed sub-tiles and reduced
    chunks leave each rank through shared-memory output tiles that TMA bulk-stores into the
    peers' receive slots / fusion buffers."""
    monkeypatch.setenv("GR_PUSH", "1")
    yield


@pytest.mark.parametrize("n", NS)
def test_virtual_push_edge_both_algorithms(gpu, n, push_mode):
    """Push path, one-shot and two-shot forced: ragged sizes, tensors spanning many chunks and
    sub-tiles (the output-tile ring wraps many times), fp16 gradients, both buffer precisions,
    integer payloads — bit-exact against oracle.emulate, replicas identical."""
    from paper_1909_11150_b200 import GR_ALGO_ONESHOT, GR_ALGO_TWOSHOT
    from tests.parity_lib import run_virtual_case
    for seed in range(2):
        rng = np.random.default_rng(100 + seed)
        T = int(rng.integers(1, 24))
        G = int(rng.integers(1, T + 1))
        numel = rng.integers(1, 200000, size=T).astype(np.int64)
        numel[rng.integers(0, T)] = int(rng.integers(1, 9))
        case = Case(n, numel, random_partition(T, G, rng), random_mark_schedule(n, T, seed, 3), seed)
        gf = (rng.random(T) < 0.3).tolist()
        for buf16 in (True, False):
            chunk = int(rng.choice([1024, 4096, 32768]))
            out = run_virtual_case(case, seed, gpu, buf16, grad_f16=gf, chunk_elems=chunk,
                                   one_shot_max_bytes=TWO_SHOT)
            assert _algos(out) == {GR_ALGO_TWOSHOT}
            out = run_virtual_case(case, seed, gpu, buf16, grad_f16=gf, chunk_elems=chunk,
                                   one_shot_max_bytes=ONE_SHOT)
            assert _algos(out) == {GR_ALGO_ONESHOT}
        run_virtual_case(case, seed, gpu, True, kind="int", one_shot_max_bytes=TWO_SHOT)
    for seed in range(4):  # configs[0]'s shape
        run_virtual_case(cfg1_case(seed, N=n), seed, gpu, seed % 2 == 0, timeout_ms=20000)


@pytest.mark.parametrize("n", [2, 4])
def test_virtual_push_numeric_edges_stats_steps(gpu, n, push_mode):
    """Push path: numeric edge cases (R8 range, subnormals, specials, cancellation) and the
    NEXT-2 statistics for both algorithms, five steps on the same contexts (receive slots and
    flags double-buffered by step parity), the fcn220m set at full size two-shot."""
    from paper_1909_11150_b200 import GR_F16, virtual_world
    from tests.parity_lib import run_case_on_rank, run_ranks, run_virtual_case
    rng = np.random.default_rng(150 + n)
    T = 7
    numel = rng.integers(1, 120000, size=T).astype(np.int64)
    case = Case(n, numel, random_partition(T, 3, rng), random_mark_schedule(n, T, 150 + n, 2), 150 + n)
    gf = [t % 3 == 0 for t in range(T)]
    for buf16 in (True, False):
        for osm in (TWO_SHOT, ONE_SHOT):
            run_virtual_case(case, 150 + n, gpu, buf16, grad_f16=gf, kind="edge", one_shot_max_bytes=osm,
                             chunk_elems=4096)
            run_virtual_case(case, 150 + n, gpu, buf16, grad_f16=gf, stats=True, one_shot_max_bytes=osm)
    base = cfg1_case(9, N=n)
    ctxs = virtual_world(world_size=n, device=0, numel=base.numel, group_of=base.group_of, buffer_dtype=GR_F16,
                         one_shot_max_bytes=TWO_SHOT, chunk_elems=256)
    try:
        for step in range(5):
            c = Case(n, base.numel, base.group_of, random_mark_schedule(n, base.T, 300 + step, 3), 300 + step)
            hs = run_ranks(n, lambda r: run_case_on_rank(ctxs[r], c, r, 300 + step, gpu, True)[1])
            assert len(set(hs)) == 1
    finally:
        for cx in ctxs:
            cx.gr_finalize()
    f = fcn220m()
    mark = reverse_layer_schedule(len(f.layers), n, f.release_order, layers_per_cycle=1, jitter_seed=n, max_shift=2)
    run_virtual_case(Case(n, f.numel, f.group_of, mark, 60 + n), 60 + n, gpu, True, one_shot_max_bytes=TWO_SHOT)


# ------------------------------------------------------------------ split queues (GR_QUEUE=1)

@pytest.mark.parametrize("n", [2, 3, 4, 8])
def test_virtual_split_queue(gpu, n, monkeypatch):
    """Split PACK / dependent queues: a producer packs while its next
    reduce-scatter / all-gather is not ready. Ragged sizes and both algorithms forced, fp16
    gradients, integer payloads, cfg1 schedules, the fcn220m set — bit-exact against
    oracle.emulate, replicas identical."""
    from paper_1909_11150_b200 import GR_ALGO_ONESHOT, GR_ALGO_TWOSHOT
    from tests.parity_lib import run_virtual_case
    monkeypatch.setenv("GR_QUEUE", "1")
    for seed in range(2):
        rng = np.random.default_rng(200 + seed)
        T = int(rng.integers(1, 24))
        G = int(rng.integers(1, T + 1))
        numel = rng.integers(1, 200000, size=T).astype(np.int64)
        case = Case(n, numel, random_partition(T, G, rng), random_mark_schedule(n, T, seed, 3), seed)
        gf = (rng.random(T) < 0.3).tolist()
        for buf16 in (True, False):
            chunk = int(rng.choice([1024, 4096, 32768]))
            out = run_virtual_case(case, seed, gpu, buf16, grad_f16=gf, chunk_elems=chunk, one_shot_max_bytes=TWO_SHOT)
            assert _algos(out) == {GR_ALGO_TWOSHOT}
            out = run_virtual_case(case, seed, gpu, buf16, grad_f16=gf, chunk_elems=chunk, one_shot_max_bytes=ONE_SHOT)
            assert _algos(out) == {GR_ALGO_ONESHOT}
        run_virtual_case(case, seed, gpu, True, kind="int", one_shot_max_bytes=TWO_SHOT)
    for seed in range(3):
        run_virtual_case(cfg1_case(seed, N=n), seed, gpu, seed % 2 == 0, timeout_ms=20000)
    if n in (2, 4):
        f = fcn220m()
        mark = reverse_layer_schedule(len(f.layers), n, f.release_order, layers_per_cycle=1, jitter_seed=n, max_shift=2)
        run_virtual_case(Case(n, f.numel, f.group_of, mark, 70 + n), 70 + n, gpu, True, one_shot_max_bytes=TWO_SHOT)


# ------------------------------------------------------------------ failure paths (§8(b) errors)

def _tiny_world(n, **kw):
    from paper_1909_11150_b200 import GR_F16, virtual_world
    return virtual_world(world_size=n, device=0, numel=[4096, 4096], group_of=[0, 1], buffer_dtype=GR_F16, **kw)


def test_virtual_rank_that_stops_stepping_times_out(gpu):
    """A rank that never enters the cycle: its peers report GR_ETIMEOUT (sticky) within about
    2 x timeout_ms (host barrier, then the device's wait on the missing LL words) instead of
    hanging; SPEC.md:406's deadlock-detection analogue."""
    import time
    import torch
    from paper_1909_11150_b200 import GrError
    from paper_1909_11150_b200.binding import GR_ESTATE, GR_ETIMEOUT
    from tests.parity_lib import run_ranks
    ctxs = _tiny_world(3, timeout_ms=400)
    x = [torch.ones(4096, device=gpu) for _ in range(6)]
    try:
        for r in range(3):
            ctxs[r].gr_mark_ready(0, x[2 * r].data_ptr())

        def rank(r):
            if r == 2:
                return None  # stalls: never calls gr_step
            t0 = time.monotonic()
            with pytest.raises(GrError) as e:
                ctxs[r].gr_step()
            assert e.value.code == GR_ETIMEOUT, e.value
            with pytest.raises(GrError) as e2:  # sticky
                ctxs[r].gr_step()
            assert e2.value.code == GR_ESTATE
            return time.monotonic() - t0

        dt = run_ranks(3, rank)
        assert all(d < 10 for d in dt[:2]), dt
        # the straggler arrives later, alone: its peers did publish cycle 0's words, so its AND
        # completes and releases group 0, but no peer ever packs: its reduction times out on
        # the peers' chunk flags (the data kernel's timeout, reported by gr_wait)
        rel, _complete, _A, _ = ctxs[2].gr_step()
        assert rel == [0]
        with pytest.raises(GrError) as e:
            ctxs[2].gr_wait()
        assert e.value.code == GR_ETIMEOUT and "reduction timed out" in str(e.value)
    finally:
        for c in ctxs:
            c.gr_finalize()


@pytest.mark.parametrize("which", ["abort", "shutdown"])
def test_virtual_status_bits_or_over_ranks(gpu, which):
    """One rank raises ABORT (or SHUTDOWN): every rank's cycle releases nothing and returns
    GR_EABORT / GR_ESHUTDOWN in the same cycle (complement-coded status bits: the one AND
    computes the OR of the flags, reading R1), A_c's status bit cleared."""
    import torch
    from paper_1909_11150_b200 import GrError
    from paper_1909_11150_b200.binding import GR_EABORT, GR_ESHUTDOWN
    from tests.parity_lib import run_ranks
    n = 4
    ctxs = _tiny_world(n, timeout_ms=5000)
    xs = [torch.ones(4096, device=gpu) for _ in range(2 * n)]
    try:
        def rank(r):
            c = ctxs[r]
            c.gr_mark_ready(0, xs[2 * r].data_ptr())
            rel, complete, A, _ = c.gr_step()  # cycle 0: group 0 released everywhere
            assert rel == [0] and not complete and (A[0] & 3) == 3
            c.gr_mark_ready(1, xs[2 * r + 1].data_ptr())
            if r == 2:
                c.gr_set_status(abort=which == "abort", shutdown=which == "shutdown")
            with pytest.raises(GrError) as e:
                c.gr_step()
            return e.value.code

        codes = run_ranks(n, rank)
        assert set(codes) == {GR_EABORT if which == "abort" else GR_ESHUTDOWN}, codes
    finally:
        for c in ctxs:
            c.gr_finalize()
