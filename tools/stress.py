"""Randomised soak test of the whole path against the oracle (one GPU): random tables, group
partitions, sizes, mark schedules, buffer precisions, fp16 gradients and payload kinds, on N=1
real contexts (armed cycles on) and N = 2/3/4/8 virtual ranks with the algorithm and the queue /
push / chunking knobs drawn at random — every case checked exactly as the parity tests do
(schedule and A_c bit-exact, values bit-exact against oracle.emulate, replicas identical).

  python tools/stress.py --minutes 10 [--seed 0]

Prints one line per case and a JSON summary; exits 1 on the first mismatch (with the case's
parameters, so it can be replayed).
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--minutes", type=float, default=10.0)
    ap.add_argument("--seed", type=int, default=0)
    a = ap.parse_args()
    import numpy as np
    import torch

    from paper_1909_11150_b200 import GR_F16, GR_F32, Context
    from tests.parity_lib import run_case_on_rank, run_virtual_case
    from workloads.schedules import Case, random_mark_schedule, random_partition

    torch.cuda.set_device(0)
    dev = torch.device("cuda", 0)
    rng = np.random.default_rng(a.seed)
    t_end = time.time() + a.minutes * 60
    n_cases = 0
    knobs_seen = {}
    while time.time() < t_end:
        seed = int(rng.integers(0, 1 << 30))
        N = int(rng.choice([1, 2, 3, 4, 8]))
        T = int(rng.integers(1, 40))
        G = int(rng.integers(1, T + 1))
        numel = rng.integers(1, int(rng.choice([64, 4096, 200000])), size=T).astype(np.int64)
        group_of = random_partition(T, G, rng)
        mark = random_mark_schedule(N, T, seed, int(rng.integers(1, 5)))
        case = Case(N, numel, group_of, mark, seed)
        buf16 = bool(rng.integers(0, 2))
        gf = (rng.random(T) < 0.25).tolist()
        kind = str(rng.choice(["uniform", "uniform", "int", "edge"]))
        env = {}
        if N > 1:
            env["GR_PUSH"] = str(int(rng.random() < 0.2))
            env["GR_QUEUE"] = str(int(rng.random() < 0.2))
            env["GR_FINE_BELOW"] = str(int(rng.choice([0, 1 << 30])))
            osm = int(rng.choice([0, 1 << 62, -1]))
            chunk = int(rng.choice([0, 0, 1024, 8192]))
        else:
            env["GR_ARM"] = "1"
            env["GR_ARM_GAP_US"] = str(int(rng.choice([50, 1 << 30])))
            env["GR_ARM_US"] = str(int(rng.choice([1, 100, 100000])))
            osm, chunk = -1, 0
        for k, v in env.items():
            os.environ[k] = v
        desc = {"seed": seed, "N": N, "T": T, "G": G, "buf16": buf16, "kind": kind, "osm": osm, "chunk": chunk, **env}
        try:
            if N == 1:
                ctx = Context(rank=0, world_size=1, device=0, numel=numel, group_of=group_of, grad_f16=gf,
                              buffer_dtype=GR_F16 if buf16 else GR_F32, timeout_ms=20000)
                try:
                    for rep in range(3):  # several steps on one context
                        run_case_on_rank(ctx, case, 0, seed + rep, dev, buf16, gf, kind)
                finally:
                    ctx.gr_finalize()
            else:
                run_virtual_case(case, seed, dev, buf16, grad_f16=gf, kind=kind, one_shot_max_bytes=osm,
                                 chunk_elems=chunk, timeout_ms=20000)
        except BaseException as e:  # noqa: BLE001 — report the case and stop
            print(json.dumps({"stress": "FAILED", "case": desc, "error": repr(e)[:2000]}), flush=True)
            sys.exit(1)
        finally:
            for k in env:
                os.environ.pop(k, None)
        n_cases += 1
        key = (N, env.get("GR_PUSH"), env.get("GR_QUEUE"))
        knobs_seen[str(key)] = knobs_seen.get(str(key), 0) + 1
        if n_cases % 25 == 0:
            print(f"{n_cases} cases ok", flush=True)
    print(json.dumps({"stress": "ok", "cases": n_cases, "minutes": a.minutes, "seed": a.seed,
                      "by_N_push_queue": knobs_seen}), flush=True)


if __name__ == "__main__":
    main()
