"""CPU tests of the boundary: libgr.so loads, exports every symbol include/gr.h
declares, validates its inputs, builds the response cache / fusion layout, and
its collective init detects cross-rank mismatches (world_size 2 over gloo).
No compute call runs here (no GPU): contexts use device = -1 ("dry")."""
import ctypes
import multiprocessing as mp
import os
import re
import socket

import numpy as np
import pytest

from tests.conftest import ROOT


def header_symbols():
    with open(os.path.join(ROOT, "include", "gr.h")) as f:
        src = f.read()
    return sorted(set(re.findall(r"^\s*(?:int|const char \*)\s*(gr_\w+)\s*\(", src, flags=re.M)))


def test_library_exports_every_declared_symbol():
    from paper_1909_11150_b200 import binding
    syms = header_symbols()
    assert len(syms) >= 12, syms
    lib = ctypes.CDLL(binding.LIB_PATH)
    for s in syms:
        assert hasattr(lib, s), f"libgr.so does not export {s}"
    assert set(syms) == set(binding.EXPORTED)


def test_library_is_sm100a_native():
    """The fatbin inside libgr.so carries sm_100a SASS (cuobjdump)."""
    import shutil
    import subprocess
    from paper_1909_11150_b200 import binding
    exe = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(exe):
        pytest.skip("cuobjdump not installed")
    out = subprocess.run([exe, "--list-elf", binding.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def dry(numel, group_of, **kw):
    from paper_1909_11150_b200 import Context
    return Context(rank=kw.pop("rank", 0), world_size=kw.pop("world_size", 1), device=-1, numel=numel,
                   group_of=group_of, **kw)


def test_dry_init_layout_matches_oracle_cache(orc):
    rng = np.random.default_rng(0)
    from workloads.schedules import random_partition
    for _ in range(50):
        T = int(rng.integers(1, 200))
        g = random_partition(T, int(rng.integers(1, T + 1)), rng)
        numel = rng.integers(1, 5000, size=T)
        ctx = dry(numel, g)
        assert ctx.W == orc.words(T)
        assert ctx.bit_of() == [int(x) for x in orc.bit_positions(g)]
        off = ctx.buf_offsets()
        # fusion layout: group-major, 8-element aligned, non-overlapping
        order = sorted(range(T), key=lambda t: (g[t], t))
        for a, b in zip(order, order[1:]):
            assert off[b] >= off[a] + numel[a] and off[b] % 8 == 0
        ctx.gr_finalize()


@pytest.mark.parametrize("T", [2046, 2047, 4096, 65536])
def test_dry_init_large_tables_match_oracle_cache(orc, T):
    """The response cache at and beyond the inline-bitvector size (W = 64 at T = 2046) up to
    cfg4's largest table: bit positions identical to the oracle's (reading R3)."""
    from workloads.schedules import random_partition
    rng = np.random.default_rng(T)
    g = random_partition(T, max(1, T // 8), rng)
    ctx = dry(np.ones(T, dtype=np.int64), g)
    assert ctx.W == orc.words(T) == (T + 2 + 31) // 32
    assert ctx.bit_of() == [int(x) for x in orc.bit_positions(g)]
    ctx.gr_finalize()


@pytest.mark.parametrize("numel,group_of", [
    ([1, 2], [0, 2]),        # group 1 empty
    ([1, 0], [0, 0]),        # numel 0
    ([1, -5], [0, 0]),       # negative
    ([4], [1]),              # G > T / id out of range
])
def test_dry_init_rejects_bad_tables(numel, group_of):
    from paper_1909_11150_b200 import GrError
    from paper_1909_11150_b200.binding import GR_EINVAL
    with pytest.raises(GrError) as e:
        dry(numel, group_of)
    assert e.value.code == GR_EINVAL


def test_dry_init_rejects_bad_world():
    from paper_1909_11150_b200 import GrError
    with pytest.raises(GrError):
        dry([8], [0], rank=3, world_size=2)
    with pytest.raises(GrError):
        dry([8], [0], chunk_elems=12)
    with pytest.raises(GrError):
        dry([8], [0], world_size=2)  # no allgather callback for N > 1
    with pytest.raises(GrError):
        dry([8], [0], world_size=9)  # one NVSwitch domain: at most 8 ranks (gr.h)
    with pytest.raises(GrError):
        dry([8], [0], world_size=0)


def test_dry_init_table_size_limit():
    """T up to ~131K tensors (the bitvector kernel's 64 KB shared-memory budget: 3 W words plus
    the complete-group mask); beyond, EINVAL. Singleton groups are the largest case."""
    from paper_1909_11150_b200 import GrError
    from paper_1909_11150_b200.binding import GR_EINVAL
    ctx = dry(np.ones(131000, dtype=np.int64), np.arange(131000))
    ctx.gr_finalize()
    with pytest.raises(GrError) as e:
        dry(np.ones(132000, dtype=np.int64), np.arange(132000))
    assert e.value.code == GR_EINVAL


def test_dry_context_refuses_compute_calls():
    from paper_1909_11150_b200 import GrError
    ctx = dry([8, 8], [0, 1])
    with pytest.raises(GrError):
        ctx.gr_mark_ready(0, 0x1000)
    with pytest.raises(GrError):
        ctx.gr_step()
    ctx.gr_finalize()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _rank_main(rank, port, mismatch, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=2)
    from paper_1909_11150_b200 import Context, GrError, make_allgather
    numel = [100, 200, 300]
    comm_ctas = 0
    if mismatch == "table" and rank == 1:
        numel = [100, 200, 301]
    if mismatch == "queue" and rank == 1:
        comm_ctas = 32  # sets the fused kernel's default queue lags: must agree across ranks
    if mismatch == "invalid" and rank == 1:
        numel = [100, 0, 300]  # rejected locally on rank 1 only: rank 0 must not hang
    try:
        ctx = Context(rank=rank, world_size=2, device=-1, numel=numel, group_of=[0, 1, 1],
                      comm_ctas=comm_ctas, allgather=make_allgather(None))
        q.put((rank, "ok", ctx.bit_of(), ctx.buf_offsets()))
        ctx.gr_finalize()
    except GrError as e:
        q.put((rank, "err", e.code, str(e)))
    dist.destroy_process_group()


@pytest.mark.parametrize("mismatch", [None, "table", "queue", "invalid"])
def test_gloo_world2_init_consistency(mismatch):
    """gr_init is collective: identical tables agree on the cache/layout;
    any difference makes gr_init fail with GR_EMISMATCH on every rank. A rank
    whose own arguments are rejected still joins the init gather, so every rank fails
    (GR_EINVAL) instead of its peers blocking."""
    from paper_1909_11150_b200.binding import GR_EINVAL, GR_EMISMATCH
    ctxm = mp.get_context("spawn")
    q = ctxm.Queue()
    port = _free_port()
    ps = [ctxm.Process(target=_rank_main, args=(r, port, mismatch, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = sorted([q.get(timeout=120) for _ in range(2)])
    for p in ps:
        p.join(60)
    if mismatch == "invalid":
        assert all(r[1] == "err" and r[2] == GR_EINVAL for r in res), res
        assert "rank 1" in res[0][3], res
    elif mismatch:
        assert all(r[1] == "err" and r[2] == GR_EMISMATCH for r in res), res
    else:
        assert all(r[1] == "ok" for r in res), res
        assert res[0][2:] == res[1][2:]


def test_plain_c_program_uses_the_abi(tmp_path):
    """The boundary is a C ABI: a C11 program compiled against include/gr.h alone and linked
    with libgr.so (no Python, no torch in that process) builds a dry context and checks the
    response cache against reading R3, the fusion layout and the error paths."""
    import shutil
    import subprocess
    if shutil.which("gcc") is None:
        pytest.skip("gcc not available")
    pkg = os.path.join(ROOT, "paper_1909_11150_b200")
    exe = str(tmp_path / "abi_dry")
    subprocess.run(["gcc", "-std=c11", "-Wall", "-Wextra", "-Werror", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "c", "abi_dry.c"), "-L", pkg, "-lgr", f"-Wl,-rpath,{pkg}",
                    "-o", exe], check=True)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=60)
    assert r.returncode == 0 and r.stdout.strip() == "ok", (r.stdout, r.stderr)


def _cuobjdump(*args):
    import shutil
    import subprocess
    exe = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(exe):
        pytest.skip("cuobjdump not installed")
    from paper_1909_11150_b200 import binding
    return subprocess.run([exe, *args, binding.LIB_PATH], capture_output=True, text=True).stdout


def test_kernel_resource_budgets():
    """The register / local-memory budgets the design relies on: no kernel
    spills to local memory; the N=1 kernel fits 4 CTAs x 256 threads per SM (<= 64 registers);
    the fused reduce kernel stays at <= 96 x 512 and the bitvector kernel at <= 64 x 256, so the
    next cycle's bitvector kernel can be resident beside a running reduction."""
    out = _cuobjdump("--dump-resource-usage")
    rows = re.findall(r"Function (\S+):\s*\n\s*REG:(\d+) STACK:(\d+) SHARED:(\d+) LOCAL:(\d+)", out)
    assert len(rows) >= 10, out[:2000]
    for name, reg, _stack, _shared, local in rows:
        reg, local = int(reg), int(local)
        assert local == 0, f"{name} uses {local} B of local memory"
        if "local_kernel" in name and "Lb0E" in name:
            assert reg <= 64, f"{name}: {reg} registers"
        if "xfer_kernel" in name:
            assert reg <= 96, f"{name}: {reg} registers"
        if "bitvector_kernel" in name:
            assert reg <= 64, f"{name}: {reg} registers"


def test_fused_reduce_kernel_uses_tma_and_multimem():
    """SASS evidence (B200_PROFILING.md mnemonics): the fused reduce kernel stages peer data with
    TMA bulk copies (UBLKCP) completed on mbarriers (SYNCS.*TRANS64) and carries the NVLS
    in-switch reduction (LDGMC = multimem.ld_reduce)."""
    sass = _cuobjdump("-sass", "-fun", "_ZN2gr11xfer_kernelI6__halfLb0EEEvNS_10DataParamsE")
    assert "UBLKCP" in sass and "SYNCS.ARRIVE.TRANS64" in sass and "LDGMC" in sass


def test_virtual_world_needs_a_device():
    """gr_init_virtual validates before touching CUDA: a dry device, world sizes outside
    2..8 and bad tables fail with GR_EINVAL and leave no contexts."""
    from paper_1909_11150_b200 import GrError, virtual_world
    from paper_1909_11150_b200.binding import GR_EINVAL
    for kw in (dict(world_size=2, device=-1), dict(world_size=1, device=0), dict(world_size=9, device=0)):
        with pytest.raises(GrError) as e:
            virtual_world(numel=[8, 8], group_of=[0, 1], **kw)
        assert e.value.code == GR_EINVAL, kw
