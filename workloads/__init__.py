"""Seeded synthetic inputs shared by tests, bench.py and smoke().

This package holds NONE of the method's arithmetic (no bitvectors, no
intersection, no release rule, no sums): only tensor tables, group
assignments, readiness (mark) schedules and gradient values, all seeded.
Both the oracle (oracle/) and the CUDA path (paper_1909_11150_b200/) consume
these inputs; neither imports the other.
"""
from .fcn import fcn220m, FcnTable  # noqa: F401
from .schedules import (  # noqa: F401
    cfg1_case,
    random_partition,
    random_mark_schedule,
    reverse_layer_schedule,
    cfg4_case,
)
from .values import grad_values  # noqa: F401
