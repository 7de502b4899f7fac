"""B200-native grouped gradient reduction (arXiv 1909.11150 §4: Bitvector
Allreduce + Grouping + fused pack / sum-allreduce / x1/N / unpack).

The product is the C-ABI library libgr.so (include/gr.h) built from csrc/ for
sm_100a; `binding` is a thin ctypes layer with the same call names. Importing
this package fails loudly when libgr.so has not been built — there is no CPU
fallback.
"""
from .binding import (  # noqa: F401
    Context,
    GrError,
    GR_F16,
    GR_F32,
    GR_ALGO_LOCAL,
    GR_ALGO_ONESHOT,
    GR_ALGO_TWOSHOT,
    gr_bench_spin,
    make_allgather,
    virtual_world,
)
