"""Thin ctypes binding over libgr.so (include/gr.h). Argument marshalling only:
every step of the method runs in the library's sm_100a kernels. The functions
keep the C names (gr_init, gr_mark_ready, gr_step, gr_wait, ...).

There is no fallback: if libgr.so is missing or fails to load, importing this
module raises.
"""
from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
# GR_LIB_PATH: load another build of the same ABI (A/B measurements of two library versions)
LIB_PATH = os.environ.get("GR_LIB_PATH") or os.path.join(_HERE, "libgr.so")

GR_OK, GR_EINVAL, GR_ESTATE, GR_EMISMATCH, GR_ECUDA, GR_ETIMEOUT, GR_EABORT, GR_ESHUTDOWN, GR_ENOMEM = \
    0, -1, -2, -3, -4, -5, -6, -7, -8
STATUS_NAMES = {0: "GR_OK", -1: "GR_EINVAL", -2: "GR_ESTATE", -3: "GR_EMISMATCH", -4: "GR_ECUDA",
                -5: "GR_ETIMEOUT", -6: "GR_EABORT", -7: "GR_ESHUTDOWN", -8: "GR_ENOMEM"}
GR_F32, GR_F16 = 0, 1
GR_Q_WORDS, GR_Q_BIT_OF, GR_Q_BUF_OFFSET, GR_Q_NCHUNKS, GR_Q_STATS, GR_Q_LAST_ALGO, GR_Q_NVLS, GR_Q_NVLS_WHY = range(8)
GR_ALGO_NONE, GR_ALGO_LOCAL, GR_ALGO_ONESHOT, GR_ALGO_TWOSHOT, GR_ALGO_NVLS = range(5)

ALLGATHER_FN = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p)


class GrWorld(ctypes.Structure):
    _fields_ = [("rank", ctypes.c_int32), ("world_size", ctypes.c_int32), ("device", ctypes.c_int32),
                ("compute_stream", ctypes.c_void_p), ("buffer_dtype", ctypes.c_int),
                ("one_shot_max_bytes", ctypes.c_int64), ("timeout_ms", ctypes.c_int32),
                ("comm_ctas", ctypes.c_int32), ("chunk_elems", ctypes.c_int64),
                ("allgather", ALLGATHER_FN), ("user", ctypes.c_void_p)]


class GrTensor(ctypes.Structure):
    _fields_ = [("numel", ctypes.c_int64), ("grad_dtype", ctypes.c_int)]


class GrCycleInfo(ctypes.Structure):
    _fields_ = [("n_released", ctypes.c_int32), ("step_complete", ctypes.c_int32), ("cycle", ctypes.c_int64),
                ("step", ctypes.c_int64), ("released_elems", ctypes.c_int64)]


class GrStats(ctypes.Structure):
    _fields_ = [("cycles", ctypes.c_int64), ("steps", ctypes.c_int64), ("bitvector_launches", ctypes.c_int64),
                ("data_launches", ctypes.c_int64), ("released_elems", ctypes.c_int64),
                ("data_kernel_ms", ctypes.c_double), ("bitvector_kernel_ms", ctypes.c_double),
                ("host_step_us", ctypes.c_double), ("host_wait_us", ctypes.c_double),
                ("bitvector_device_us", ctypes.c_double), ("data_launches_skipped", ctypes.c_int64),
                ("armed_cycles", ctypes.c_int64), ("armed_expired", ctypes.c_int64)]


class GrError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"{STATUS_NAMES.get(code, code)}: {msg}")
        self.code = code


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: run `python -c 'import __graft_entry__ as g; g.build()'` "
                          "(there is no CPU fallback)")
    L = ctypes.CDLL(LIB_PATH)
    p, i32, i64 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64
    sig = {
        "gr_init": ([ctypes.POINTER(p), ctypes.POINTER(GrWorld), ctypes.POINTER(GrTensor), i32, p, i32], ctypes.c_int),
        "gr_init_virtual": ([p, ctypes.POINTER(GrWorld), ctypes.POINTER(GrTensor), i32, p, i32], ctypes.c_int),
        "gr_mark_ready": ([p, i32, i32, p], ctypes.c_int),
        "gr_mark_ready_async": ([p, i32, i32, p, p], ctypes.c_int),
        "gr_mark_ready_batch": ([p, i32, i32, p, p], ctypes.c_int),
        "gr_step": ([p, p, ctypes.POINTER(GrCycleInfo), p], ctypes.c_int),
        "gr_wait": ([p], ctypes.c_int),
        "gr_wait_async": ([p], ctypes.c_int),
        "gr_released_wait_async": ([p, p], ctypes.c_int),
        "gr_step_drain": ([p], ctypes.c_int),
        "gr_set_status": ([p, i32, i32], ctypes.c_int),
        "gr_finalize": ([p], ctypes.c_int),
        "gr_last_error": ([p], ctypes.c_char_p),
        "gr_query": ([p, i32, p, ctypes.c_size_t], ctypes.c_int),
        "gr_set_timing": ([p, i32], ctypes.c_int),
        "gr_reset_stats": ([p], ctypes.c_int),
        "gr_bench_spin": ([i64, i32, p], ctypes.c_int),
        "gr_enable_grad_stats": ([p, i32], ctypes.c_int),
        "gr_grad_stats": ([p, p, p, p, p], ctypes.c_int),
    }
    for name, (args, res) in sig.items():
        f = getattr(L, name)
        f.argtypes = args
        f.restype = res
    return L


lib = _load()
EXPORTED = ("gr_init", "gr_init_virtual", "gr_mark_ready", "gr_mark_ready_batch", "gr_mark_ready_async", "gr_step", "gr_wait", "gr_wait_async", "gr_released_wait_async", "gr_step_drain", "gr_set_status",
            "gr_finalize", "gr_last_error", "gr_query", "gr_set_timing", "gr_reset_stats", "gr_bench_spin",
            "gr_enable_grad_stats", "gr_grad_stats")


def _check(rc: int, ctx=None):
    if rc != GR_OK:
        raise GrError(rc, lib.gr_last_error(ctx).decode())
    return rc


def make_allgather(pg=None, device=None):
    """Allgather callback over torch.distributed (gloo: CPU tensors, nccl: CUDA tensors)."""
    import torch
    import torch.distributed as dist

    def cb(send, recv, nbytes, _user):
        try:
            ws = dist.get_world_size(pg)
            backend = dist.get_backend(pg)
            dev = torch.device("cuda", device) if (backend == "nccl" and device is not None) else \
                (torch.device("cuda", torch.cuda.current_device()) if backend == "nccl" else torch.device("cpu"))
            src = torch.frombuffer(bytearray(ctypes.string_at(send, nbytes)), dtype=torch.uint8).to(dev)
            out = torch.empty(ws * nbytes, dtype=torch.uint8, device=dev)
            dist.all_gather_into_tensor(out, src, group=pg)
            data = out.cpu().numpy().tobytes()
            ctypes.memmove(recv, data, len(data))
            return 0
        except Exception as e:  # never raise through the C frame
            print(f"[gr allgather] {e!r}")
            return 1

    return ALLGATHER_FN(cb)


def _tables(numel, group_of, grad_f16):
    T = len(numel)
    tab = (GrTensor * T)()
    for t in range(T):
        tab[t].numel = int(numel[t])
        tab[t].grad_dtype = GR_F16 if (grad_f16 is not None and grad_f16[t]) else GR_F32
    grp = (ctypes.c_int32 * T)(*[int(g) for g in group_of])
    return T, int(max(group_of)) + 1, tab, grp


class Context:
    """Owns one gr_ctx; methods map 1:1 onto the C calls."""

    def __init__(self, *, rank: int, world_size: int, device: int, numel, group_of, grad_f16=None,
                 buffer_dtype: int = GR_F16, compute_stream: int = 0, one_shot_max_bytes: int = -1,
                 timeout_ms: int = 0, comm_ctas: int = 0, chunk_elems: int = 0, allgather=None, _handle=None):
        T, G, tab, grp = _tables(numel, group_of, grad_f16)
        self.T, self.G = T, G
        if _handle is not None:  # one rank of gr_init_virtual (virtual_world)
            self._ctx = ctypes.c_void_p(_handle)
        else:
            self._allgather = allgather if allgather is not None else ALLGATHER_FN()
            w = GrWorld(rank, world_size, device, compute_stream, buffer_dtype, one_shot_max_bytes, timeout_ms,
                        comm_ctas, chunk_elems, self._allgather, None)
            self._ctx = ctypes.c_void_p()
            rc = lib.gr_init(ctypes.byref(self._ctx), ctypes.byref(w), tab, T, ctypes.cast(grp, ctypes.c_void_p), G)
            _check(rc, None)
        self.rank = rank
        self.W = self.query_int(GR_Q_WORDS)
        self._released = (ctypes.c_int32 * self.G)()
        self._bits = (ctypes.c_uint32 * self.W)()
        self._info = GrCycleInfo()
        # marshalled once: a ctypes.cast costs ~1-2 us, a measurable part of a ~10 us cycle
        self._released_p = ctypes.cast(self._released, ctypes.c_void_p)
        self._bits_p = ctypes.cast(self._bits, ctypes.c_void_p)
        self._info_p = ctypes.byref(self._info)

    # -- the four calls of the method ------------------------------------------------------
    def gr_mark_ready(self, tensor_id: int, dev_ptr: int, rank: int | None = None):
        return _check(lib.gr_mark_ready(self._ctx, self.rank if rank is None else rank, tensor_id, dev_ptr), self._ctx)

    def gr_mark_ready_batch(self, tensor_ids, dev_ptrs, rank: int | None = None):
        n = len(tensor_ids)
        ids = (ctypes.c_int32 * n)(*tensor_ids)
        ptrs = (ctypes.c_void_p * n)(*dev_ptrs)
        return _check(lib.gr_mark_ready_batch(self._ctx, self.rank if rank is None else rank, n,
                                              ctypes.cast(ids, ctypes.c_void_p), ctypes.cast(ptrs, ctypes.c_void_p)),
                      self._ctx)

    def prepare_batch(self, tensor_ids, dev_ptrs):
        """Pre-marshalled arguments for repeated gr_mark_ready_batch calls (hot loops)."""
        n = len(tensor_ids)
        return (n, (ctypes.c_int32 * n)(*tensor_ids), (ctypes.c_void_p * n)(*dev_ptrs))

    def gr_mark_ready_prepared(self, batch, rank: int | None = None):
        n, ids, ptrs = batch
        return _check(lib.gr_mark_ready_batch(self._ctx, self.rank if rank is None else rank, n, ids, ptrs), self._ctx)

    def gr_mark_ready_async(self, tensor_id: int, dev_ptr: int, stream: int, rank: int | None = None):
        return _check(lib.gr_mark_ready_async(self._ctx, self.rank if rank is None else rank, tensor_id, dev_ptr,
                                              stream), self._ctx)

    def gr_step(self, bits: bool = True):
        """Returns (released group ids, step_complete, A words (list of int, or None when
        bits=False: skips copying W words into a Python list), info)."""
        rc = lib.gr_step(self._ctx, self._released_p, self._info_p, self._bits_p if bits else None)
        if rc:
            _check(rc, self._ctx)
        n = self._info.n_released
        return self._released[:n], bool(self._info.step_complete), (list(self._bits) if bits else None), self._info

    def gr_wait(self):
        return _check(lib.gr_wait(self._ctx), self._ctx)

    def gr_wait_async(self):
        return _check(lib.gr_wait_async(self._ctx), self._ctx)

    def gr_step_drain(self):
        """Final, device-driven cycle of the step (every tensor already marked); the host does
        not wait. Follow with gr_wait / gr_wait_async."""
        return _check(lib.gr_step_drain(self._ctx), self._ctx)

    def gr_released_wait_async(self, stream: int = 0):
        """`stream` (a raw cudaStream_t; 0 = the compute stream) waits for every group released
        so far in this step."""
        return _check(lib.gr_released_wait_async(self._ctx, ctypes.c_void_p(stream or None)), self._ctx)

    # -- extras ------------------------------------------------------------------------------
    def gr_set_status(self, abort: bool = False, shutdown: bool = False):
        return _check(lib.gr_set_status(self._ctx, int(abort), int(shutdown)), self._ctx)

    def query_int(self, kind: int) -> int:
        v = ctypes.c_int32()
        _check(lib.gr_query(self._ctx, kind, ctypes.byref(v), 4), self._ctx)
        return v.value

    def bit_of(self):
        a = (ctypes.c_int32 * self.T)()
        _check(lib.gr_query(self._ctx, GR_Q_BIT_OF, a, 4 * self.T), self._ctx)
        return list(a)

    def buf_offsets(self):
        a = (ctypes.c_int64 * self.T)()
        _check(lib.gr_query(self._ctx, GR_Q_BUF_OFFSET, a, 8 * self.T), self._ctx)
        return list(a)

    def nvls(self):
        """(enabled, reason) of the NVLS multicast path."""
        buf = ctypes.create_string_buffer(256)
        _check(lib.gr_query(self._ctx, GR_Q_NVLS_WHY, buf, 256), self._ctx)
        return self.query_int(GR_Q_NVLS) == 1, buf.value.decode()

    def stats(self) -> GrStats:
        s = GrStats()
        _check(lib.gr_query(self._ctx, GR_Q_STATS, ctypes.byref(s), ctypes.sizeof(s)), self._ctx)
        return s

    def gr_enable_grad_stats(self, on: bool = True):
        return _check(lib.gr_enable_grad_stats(self._ctx, int(on)), self._ctx)

    def gr_grad_stats(self):
        """(sum of squares per tensor [list of float], non-finite flag) of the last step."""
        ss = (ctypes.c_double * self.T)()
        nf = ctypes.c_int32()
        _check(lib.gr_grad_stats(self._ctx, ctypes.cast(ss, ctypes.c_void_p), ctypes.byref(nf), None, None),
               self._ctx)
        return list(ss), bool(nf.value)

    def set_timing(self, on: bool):
        _check(lib.gr_set_timing(self._ctx, int(on)), self._ctx)

    def reset_stats(self):
        _check(lib.gr_reset_stats(self._ctx), self._ctx)

    def last_error(self) -> str:
        return lib.gr_last_error(self._ctx).decode()

    def gr_finalize(self):
        if self._ctx:
            lib.gr_finalize(self._ctx)
            self._ctx = ctypes.c_void_p()

    def __del__(self):
        try:
            self.gr_finalize()
        except Exception:
            pass


def virtual_world(*, world_size: int, device: int, numel, group_of, grad_f16=None, buffer_dtype: int = GR_F16,
                  compute_stream: int = 0, one_shot_max_bytes: int = -1, timeout_ms: int = 0, comm_ctas: int = 0,
                  chunk_elems: int = 0):
    """gr_init_virtual: world_size ranks on one device, one Context per rank. Their collective
    calls (gr_step, gr_step_drain) must be made concurrently, one thread per rank (ctypes
    releases the GIL during the call)."""
    T, G, tab, grp = _tables(numel, group_of, grad_f16)
    w = GrWorld(0, world_size, device, compute_stream, buffer_dtype, one_shot_max_bytes, timeout_ms, comm_ctas,
                chunk_elems, ALLGATHER_FN(), None)
    outs = (ctypes.c_void_p * world_size)()
    _check(lib.gr_init_virtual(ctypes.cast(outs, ctypes.c_void_p), ctypes.byref(w), tab, T,
                               ctypes.cast(grp, ctypes.c_void_p), G), None)
    return [Context(rank=r, world_size=world_size, device=device, numel=numel, group_of=group_of, grad_f16=grad_f16,
                    _handle=outs[r]) for r in range(world_size)]


def gr_bench_spin(ns: int, ctas: int, stream: int):
    return _check(lib.gr_bench_spin(int(ns), int(ctas), stream))
