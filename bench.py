"""bench.py — grouped gradient reduction (arXiv 1909.11150 §4) on B200.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
  N>1: python -m torch.distributed.run --nnodes=1 --nproc-per-node N \
           --master-addr 127.0.0.1 --master-port P bench.py --gpus N ...

Workload (BASELINE.json configs[1] at N=1, configs[2] at N>1): the fcn220m
gradient set (68 fp32 tensors, 225,115,137 elements,
10 per-level groups), fp16 fusion buffer. One bench STEP is one pass of the
whole hot path over one step's gradients: gr_mark_ready for all 68 tensors
(reverse-layer order) -> gr_step (bitvector populate/AND/release: all 10
groups complete and are fused into one message) -> fused
pack -> sum-allreduce -> x1/N -> unpack -> gr_wait. Inputs are resident in
HBM (900 MB per rank > 126 MB L2, so no L2 flush is needed).

value = whole-job reduced-gradient throughput = N * E * 4 B / t_step (GB/s,
weak scaling: each rank reduces its own full gradient set). Per-rank NVLink
bus bandwidth (NCCL-tests convention, S*2(N-1)/N / t) is `busbw_GBps`.
Also reported: exposed communication per step with a synthetic backward
(cfg3), the bitvector cycle latency, NCCL all_reduce on the same fused
buffer (N>1), the roofline of the dominant kernel and the CPU oracle.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "grouped grad allreduce bus GB/s & exposed comm ms/step at 1/2/4/8 B200"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--buffer", default="f16", choices=["f16", "f32"])
    ap.add_argument("--exposed-steps", type=int, default=6)
    ap.add_argument("--cycle-us", type=float, default=250.0)
    ap.add_argument("--comm-sms", type=int, default=16)
    ap.add_argument("--no-extras", action="store_true", help="skip exposed-comm / cycle / NCCL / CPU legs")
    ap.add_argument("--exposed-sweep", default="",
                    help="cfg3 sweep only: 'cycle_us:comm_sms,...' pairs, one JSON line each, then exit")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    return ap.parse_args()


# ------------------------------------------------------------------ clocks sampling
class ClockSampler:
    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.path = os.path.join(ROOT, "gpurun_out", f"clocks_rank{gpu_index}_{os.getpid()}.csv")
        self.t_timed_end = None

    def __enter__(self):
        os.makedirs(os.path.dirname(self.path), exist_ok=True)
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.f = open(self.path, "w")
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "50"],
                                         stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None
        time.sleep(0.3)
        self.t_start = time.time()
        return self

    def mark_timed_end(self):
        self.t_timed_end = time.time()

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            self.proc.wait()
            self.f.close()

    def summary(self):
        try:
            rows = [l.split(",") for l in open(self.path) if l.strip()]
        except Exception:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[1]) for r in rows if len(r) >= 9 and r[1].strip().replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if len(r) >= 9 and r[2].strip().replace(".", "").isdigit()]
        reasons = set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in rows:
            if len(r) < 9:
                continue
            for n, v in zip(names, r[5:9]):
                if v.strip() == "Active":
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(rows),
                "window": "timed region + 1 s soak of the identical step (nvidia-smi -lms 50)"}


# ------------------------------------------------------------------ CPU oracle leg
def cpu_oracle_leg(N: int, seconds: float, buffer_f16: bool):
    """The oracle (oracle/, single-threaded C) on a bounded sample of the same
    workload: the full fcn220m schedule simulation plus the fp64 reference and
    the exact rank-order emulation on a prefix sample of every tensor."""
    import numpy as np

    import oracle
    from workloads import fcn220m
    from workloads.values import tensor_scales, values_np

    f = fcn220m()
    frac = 1.0 / 64
    s = tensor_scales(1, f.T)
    samples = []
    for t in range(f.T):
        n = max(1, int(f.numel[t] * frac))
        samples.append([values_np(1, r, t, np.arange(n), float(s[t])) for r in range(N)])
    n_elems = sum(x[0].size for x in samples)
    mark = np.zeros((N, f.T), np.int32)  # bench step: every tensor marked before cycle 0
    reps = 0
    t0 = time.perf_counter()
    while True:
        oracle.simulate_step(N, f.group_of, mark, max_cycles=4)
        for gs in samples:
            oracle.reduce_f64(gs)
            oracle.emulate(gs, buffer_f16, False)
        reps += 1
        if time.perf_counter() - t0 >= seconds:
            break
    dt = (time.perf_counter() - t0) / reps
    gbs = N * n_elems * 4 / dt / 1e9
    return {"value": round(gbs, 4), "unit": "GB/s", "cores": 1, "kind": "oracle",
            "sample": f"fcn220m schedule (68 tensors, 10 groups) + fp64 reduce and exact emulation of a "
                      f"1/64 prefix of every tensor ({n_elems} elements x {N} ranks), {reps} reps, "
                      f"{dt * 1e3:.1f} ms/rep, host nproc={os.cpu_count()}",
            "seconds_per_step_sample": dt}


def run_reference(args):
    """--impl reference: the oracle as it stands, timed on host cores, same metric/unit."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    N = args.gpus
    warm = max(0, args.warmup)
    per = max(0.5, min(6.0, 150.0 / max(1, args.steps + warm)))
    for _ in range(min(warm, 2)):
        cpu_oracle_leg(N, 0.2, args.buffer == "f16")
    times = []
    last = None
    for _ in range(args.steps):
        last = cpu_oracle_leg(N, per * 0.2, args.buffer == "f16")
        times.append(last["seconds_per_step_sample"])
    v = last["value"] if last else None
    ms = statistics.mean(times) * 1e3 if times else None
    out = {"impl": "reference", "metric": METRIC, "value": v, "unit": "GB/s", "n_gpus": N, "steps": args.steps,
           "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
           "vs_baseline": None, "dtype": "f64", "data": "synthetic",
           # the same workload as our arm (its config keys); each timed step is a bounded sample
           # of it (1/64 of every tensor, the schedule in full), described in cpu_baseline.sample
           "config": {"workload": "fcn220m_cfg2_pack_scale_unpack" if N == 1 else "fcn220m_cfg3_bitvector_grouping",
                      "tensors": 68, "groups": 10, "elements": 225115137, "buffer": args.buffer,
                      "sampled_fraction": 1 / 64},
           "cpu_baseline": {k: last[k] for k in ("value", "unit", "cores", "kind", "sample")} if last else None,
           "e2e": {"value": v, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


def nvlink_read(index: int):
    try:
        sys.path.insert(0, os.path.join(ROOT, "tools"))
        import nvlink_counters
        return nvlink_counters.read(index)
    except Exception as e:  # noqa: BLE001 — the counters are evidence, not the measurement
        return {"error": repr(e)}


def nvlink_summary(a, b, steps: int, S: int, N: int, dev):
    """Per-GPU NVLink bytes per step from NVML's cumulative counters, gathered from every rank,
    set against the algorithmic 2(N-1)/N*S per direction (two-shot / one-shot at N=2)."""
    import torch
    import torch.distributed as dist
    keys = ("tx", "rx")
    row = []
    for k in keys:
        ok = isinstance(a, dict) and isinstance(b, dict) and a.get(k) is not None and b.get(k) is not None
        row.append(float(b[k] - a[k]) / steps if ok else -1.0)
    t = torch.tensor(row, dtype=torch.float64, device=dev)
    allr = [torch.empty_like(t) for _ in range(N)]
    dist.all_gather(allr, t)
    per_rank = [[None if x < 0 else x for x in r.tolist()] for r in allr]
    alg = 2 * (N - 1) / N * S
    return {"per_rank_per_step": [dict(zip(keys, r)) for r in per_rank],
            "units": "bytes: nvidia-smi nvlink -gt d (data Tx/Rx, summed over links) per step",
            "ratio_tx_over_algorithmic": [None if r[0] is None else round(r[0] / alg, 4) for r in per_rank],
            "ratio_rx_over_algorithmic": [None if r[1] is None else round(r[1] / alg, 4) for r in per_rank],
            "algorithmic_bytes_per_direction_per_step": alg, "steps": steps,
            "note": "counter scale checked by tools/nvlink_counters.py (peer copy of a known size)"}


def _max_over(x: float, dev) -> float:
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


# ------------------------------------------------------------------ our arm
def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
        return

    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_1909_11150_b200 as gr
    from workloads import fcn220m
    from workloads.values import fill_values_torch, tensor_scales

    rank = int(os.environ.get("RANK", "0"))
    N = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    assert N == args.gpus, f"--gpus {args.gpus} but WORLD_SIZE={N}"
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if N > 1:
        dist.init_process_group("nccl", device_id=dev)
    compute = torch.cuda.current_stream(dev)
    props = torch.cuda.get_device_properties(dev)
    sms = props.multi_processor_count

    f = fcn220m()
    E = int(f.numel.sum())
    buf16 = args.buffer == "f16"
    pb = 2 if buf16 else 4
    s = tensor_scales(1, f.T)
    grads = []
    for t in range(f.T):
        x = torch.empty(int(f.numel[t]), dtype=torch.float32, device=dev)
        fill_values_torch(x, 1, rank, t, float(s[t]))
        grads.append(x)
    ptrs = [g.data_ptr() for g in grads]
    tensor_order = [t for l in f.release_order for t in (2 * l, 2 * l + 1)]
    torch.cuda.synchronize()

    ag = gr.make_allgather(None, local) if N > 1 else None
    ctx = gr.Context(rank=rank, world_size=N, device=local, numel=f.numel, group_of=f.group_of,
                     buffer_dtype=gr.GR_F16 if buf16 else gr.GR_F32, compute_stream=compute.cuda_stream,
                     timeout_ms=30000, allgather=ag)

    def barrier():
        if N > 1:
            dist.barrier(device_ids=[local])

    if args.exposed_sweep:  # cfg3 sweep of the cycle time and of the SMs given to communication
        for pair in args.exposed_sweep.split(","):
            cu, cs = pair.split(":")
            r = exposed_comm(args, float(cu), int(cs), f, ptrs, N, rank, local, dev, compute, sms, barrier,
                             lambda x: x if N == 1 else _max_over(x, dev), gr)
            if rank == 0:
                print(json.dumps({"cfg3_sweep": True, "n_gpus": N, **r["exposed_comm"]}), flush=True)
        ctx.gr_finalize()
        return

    batch = ctx.prepare_batch(tensor_order, [ptrs[t] for t in tensor_order])

    def one_step(blocking=False):
        ctx.gr_mark_ready_prepared(batch)  # all 68 tensors, reverse-layer order, one call
        rel, complete, _A, _ = ctx.gr_step()
        assert complete and len(rel) == f.G, (rel, complete)
        if blocking:
            ctx.gr_wait()        # host blocks until the reduction is done
        else:
            ctx.gr_wait_async()  # stream-ordered: compute_stream waits, the host moves on

    def max_over_ranks(x: float) -> float:
        if N == 1:
            return x
        tt = torch.tensor([x], dtype=torch.float64, device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        return float(tt.item())

    # ---- headline: device-timed K steps ----
    for _ in range(max(3, args.warmup)):
        one_step()
    ctx.reset_stats()
    barrier()
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        ev0.record(compute)
        for _ in range(args.steps):
            one_step()
        ev1.record(compute)
        torch.cuda.synchronize()
        st_timed = ctx.stats()
        clk.mark_timed_end()
        ms_local = ev0.elapsed_time(ev1) / args.steps
        # the timed region is often far shorter than nvidia-smi's sampling period: keep the
        # identical step running (untimed) for ~1 s so the clock record covers this load. The
        # step count comes from the max-over-ranks time, so every rank runs the same number of
        # collective steps.
        n_soak = int(min(20000, max(1, 1000.0 / max(1e-3, max_over_ranks(ms_local)))))
        nvl0 = nvlink_read(local) if N > 1 else None
        for _ in range(n_soak):
            one_step()
        torch.cuda.synchronize()
        nvl1 = nvlink_read(local) if N > 1 else None
    barrier()
    st = st_timed  # counters of exactly the K timed steps (the clock soak follows)
    ctx_nvls = "%s (%s)" % ctx.nvls() if N > 1 else None
    # the same steps with a host-blocking gr_wait (host latency exposed every step)
    ev2, ev3 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    nb = max(3, min(args.steps, 20))
    barrier()
    torch.cuda.synchronize()
    ev2.record(compute)
    for _ in range(nb):
        one_step(blocking=True)
    ev3.record(compute)
    torch.cuda.synchronize()
    ms_blocking = max_over_ranks(ev2.elapsed_time(ev3) / nb)
    ms = max_over_ranks(ms_local)
    launches = int(st.bitvector_launches + st.data_launches)
    algo = ctx.query_int(gr.binding.GR_Q_LAST_ALGO)
    value = N * E * 4 / (ms * 1e-3) / 1e9
    S = E * pb
    busbw = (S / (ms * 1e-3) * 2 * (N - 1) / N / 1e9) if N > 1 else None

    # ---- dominant kernel timing (CUDA events on the library's own data stream) ----
    ctx.set_timing(True)
    ctx.reset_stats()
    for _ in range(max(3, min(args.steps, 10))):
        one_step(blocking=True)  # blocking wait collects the per-launch event timings
    stt = ctx.stats()
    ctx.set_timing(False)
    kern_ms = stt.data_kernel_ms / max(1, stt.data_launches)
    bv_ms = stt.bitvector_kernel_ms / max(1, stt.bitvector_launches)
    kern_ms = max_over_ranks(kern_ms)
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        pass
    if N == 1:
        alg_bytes = E * 8  # LOCAL: read fp32 g, write fp32 g (the fusion buffer is elided at N=1)
        hbm = peaks.get("hbm_gbs")
        roof = {"bound": "hbm", "achieved": round(alg_bytes / (kern_ms * 1e-3) / 1e9, 1),
                "peak": hbm if hbm else 6650.0, "unit": "GB/s",
                "peak_source": "MEASURED_PEAKS.json hbm_gbs" if hbm else "B200_PROFILING.md fallback",
                "kernel": f"local_kernel<{'half' if buf16 else 'float'}>", "algorithmic_bytes_per_launch": alg_bytes,
                "kernel_ms": round(kern_ms, 4),
                # SURVEY.md §8(d) cfg2 counts pack (p_g+p_b) + unpack (p_b+p_g) through a materialised
                # fusion buffer: 12 B/elem at fp16. At N=1 no peer reads the buffer, so the kernel
                # fuses pack->x1/N->unpack in registers (8 B/elem, bit-identical): on the survey's
                # count the same kernel would read above 1 of peak, i.e. the buffer is not moved.
                "survey_cfg2_bytes_per_elem": 2 * (4 + pb),
                "frac_on_survey_bytes": round(E * 2 * (4 + pb) / (kern_ms * 1e-3) / 1e9 / (hbm if hbm else 6650.0), 4)}
    else:
        alg_bytes = int(2 * (N - 1) / N * S)  # bytes that must cross NVLink per direction per rank
        roof = {"bound": "nvlink", "achieved": round(alg_bytes / (kern_ms * 1e-3) / 1e9, 1), "peak": 770.0,
                "unit": "GB/s", "peak_source": "B200_PROFILING.md measured peer copy per direction (900 nominal)",
                "kernel": f"xfer_kernel<{'half' if buf16 else 'float'}>:{ {2: 'ONESHOT', 3: 'TWOSHOT', 4: 'NVLS'}.get(algo) }",
                "algorithmic_bytes_per_launch": alg_bytes, "kernel_ms": round(kern_ms, 4),
                "peak_north_star": 900.0,
                "frac_of_north_star_900": round(alg_bytes / (kern_ms * 1e-3) / 1e9 / 900.0, 4)}
    roof["frac"] = round(roof["achieved"] / roof["peak"], 4)
    roof["traffic"] = None
    try:
        prof = json.load(open(os.path.join(ROOT, "profiles", "traffic.json")))
        key = f"N{N}_{args.buffer}"
        if key in prof:
            roof["traffic"] = prof[key]["dram_bytes_per_launch"]
            roof["traffic_source"] = prof[key]["source"]
    except Exception:
        pass

    extras = {}
    if not args.no_extras:
        extras = run_extras(args, ctx, grads, ptrs, tensor_order, f, N, rank, local, dev, compute, sms, barrier,
                            max_over_ranks, gr)

    # ---- e2e: host buffers, H2D + step + D2H inside the timed region ----
    # Through the public API the way a host-fed job would use it: each tensor is copied in on a
    # copy stream and marked ready stream-ordered right behind its copy (gr_mark_ready_async);
    # coordination cycles run while the copies stream in, each released group is copied back
    # out as soon as its reduction is done (gr_released_wait_async on a second copy stream).
    host_in = [torch.empty(g.numel(), dtype=torch.float32, pin_memory=True) for g in grads]
    host_out = [torch.empty(g.numel(), dtype=torch.float32, pin_memory=True) for g in grads]
    for h, g in zip(host_in, grads):
        h.copy_(g)
    s_in, s_out = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
    tensors_of = {}
    for t in range(f.T):
        tensors_of.setdefault(int(f.group_of[t]), []).append(t)
    e2e_steps = max(2, min(args.steps, 4))

    def e2e_step():
        s_in.wait_stream(compute)   # previous step's reduction and copy-out are done
        s_in.wait_stream(s_out)
        with torch.cuda.stream(s_in):
            for t in tensor_order:
                grads[t].copy_(host_in[t], non_blocking=True)
                ctx.gr_mark_ready_async(t, ptrs[t], s_in.cuda_stream)
        complete, cycles = False, 0
        while not complete:
            rel, complete, _A, _ = ctx.gr_step(bits=False)
            cycles += 1
            if rel:
                ctx.gr_released_wait_async(s_out.cuda_stream)
                with torch.cuda.stream(s_out):
                    for g in rel:
                        for t in tensors_of[g]:
                            host_out[t].copy_(grads[t], non_blocking=True)
            elif not complete:
                t_next = time.perf_counter() + 50e-6  # 50 us cycle time while nothing is ready
                while time.perf_counter() < t_next:
                    pass
        ctx.gr_wait_async()
        compute.wait_stream(s_out)
        return cycles

    e2e_step()  # warm-up of the pipelined path
    torch.cuda.synchronize()
    barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(compute)
    e2e_cycles = 0
    for _ in range(e2e_steps):
        e2e_cycles += e2e_step()
    e1.record(compute)
    torch.cuda.synchronize()
    e2e_ms = max_over_ranks(e0.elapsed_time(e1) / e2e_steps)
    ok_vals = all(torch.equal(host_out[t][:64], grads[t][:64].cpu()) for t in (0, f.T // 2, f.T - 1))
    # the same bytes moved serially (all copies in, one step, all copies out) for comparison
    barrier()
    torch.cuda.synchronize()
    e2, e3 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e2.record(compute)
    for _ in range(e2e_steps):
        for h, g in zip(host_in, grads):
            g.copy_(h, non_blocking=True)
        one_step()
        for h, g in zip(host_out, grads):
            h.copy_(g, non_blocking=True)
    e3.record(compute)
    torch.cuda.synchronize()
    e2e_serial_ms = max_over_ranks(e2.elapsed_time(e3) / e2e_steps)
    e2e = {"value": round(N * E * 4 / (e2e_ms * 1e-3) / 1e9, 3), "unit": "GB/s", "ms_per_step": round(e2e_ms, 3),
           "h2d_bytes_per_step": E * 4, "d2h_bytes_per_step": E * 4,
           "how": "pinned host -> device copies marked ready stream-ordered per tensor; cycles every <=50 us; "
                  "each released group copied back as soon as reduced (gr_released_wait_async)",
           "cycles_per_step": e2e_cycles / e2e_steps, "copy_out_matches_device": ok_vals,
           "serial_ms_per_step": round(e2e_serial_ms, 3)}

    cpu = None
    if rank == 0 and N == 1 and not args.no_extras:
        cpu = cpu_oracle_leg(N, args.cpu_seconds, buf16)
        cpu.pop("seconds_per_step_sample", None)

    nvlink = None
    if N > 1:  # NVLink payload counters over the soak's identical steps, per step, vs 2(N-1)/N*S
        nvlink = nvlink_summary(nvl0, nvl1, n_soak, S, N, dev)
    if rank == 0:
        out = {"metric": METRIC, "value": round(value, 3), "unit": "GB/s", "n_gpus": N, "steps": args.steps,
               "warmup": args.warmup, "ms_per_step": round(ms, 4), "higher_is_better": True, "scaling": "weak",
               "vs_baseline": None, "dtype": "f32", "wire_dtype": "f16" if buf16 else "f32",
               "dtype_note": "fp32 gradients, fp32 accumulation; the fusion buffer / NVLink wire holds fp16 (RN-even) with --buffer f16",
               "data": "synthetic (counter-based seeded fp32 gradients; fcn220m shapes, SURVEY.md App. A)",
               "config": {"workload": "fcn220m_cfg2_pack_scale_unpack" if N == 1 else "fcn220m_cfg3_bitvector_grouping",
                          "tensors": f.T, "groups": f.G, "elements": E, "buffer": args.buffer,
                          "message_bytes": S, "algo": {1: "local", 2: "one-shot", 3: "two-shot", 4: "nvls"}.get(algo),
                          "l2": "inputs 900 MB/rank > 126 MB L2 (no flush needed)",
                          "nvls": ctx_nvls,
                          "step": "mark 68 -> gr_step (1 cycle, 10 groups fused) -> pack/reduce/unpack -> gr_wait"},
               "value_is": "aggregate reduced-gradient GB/s = N*E*4B/t_step; per-rank NVLink bus GB/s in busbw_GBps",
               "busbw_GBps": round(busbw, 2) if busbw else None,
               "wait": "gr_wait_async (stream-ordered; the production contract)",
               "ms_per_step_blocking_wait": round(ms_blocking, 4),
               "gpu_launches": launches, "launches_per_step": launches / args.steps,
               "armed_cycles": int(st.armed_cycles), "armed_expired": int(st.armed_expired),
               "bitvector_kernel_us": round(bv_ms * 1e3, 2),
               "roofline": roof, "clocks": clk.summary(), "e2e": e2e, "cpu_baseline": cpu}
        if nvlink is not None:
            out["nvlink_counters"] = nvlink
        out.update(extras)
        print(json.dumps(out), flush=True)
    ctx.gr_finalize()
    if N > 1:
        dist.destroy_process_group()


def exposed_comm(args, cycle_us, comm_sms, f, ptrs, N, rank, local, dev, compute, sms, barrier, max_over_ranks, gr):
    """cfg3: exposed communication behind a synthetic backward pass. Reported
    two ways: SURVEY's definition max_r end of comm - max_r end of backward (the headline
    `exposed_comm_ms`; the start events follow a barrier + device sync on every rank), and per
    rank (own end of comm - own end of backward, then max / mean over ranks; it also counts a
    fast rank waiting for the slowest rank's backward)."""
    import numpy as np
    import torch
    import torch.distributed as dist

    ctx2 = gr.Context(rank=rank, world_size=N, device=local, numel=f.numel, group_of=f.group_of,
                      buffer_dtype=gr.GR_F16 if args.buffer == "f16" else gr.GR_F32,
                      compute_stream=compute.cuda_stream, timeout_ms=30000, comm_ctas=comm_sms,
                      allgather=gr.make_allgather(None, local) if N > 1 else None)
    cyc = cycle_us * 1e-6
    exposed, bwd, survey = [], [], []
    for step in range(args.exposed_steps + 2):
        rng = np.random.default_rng(1000003 * step + rank)
        barrier()
        torch.cuda.synchronize()
        ev_start = torch.cuda.Event(enable_timing=True)
        ev_bwd = torch.cuda.Event(enable_timing=True)
        ev_end = torch.cuda.Event(enable_timing=True)
        ev_start.record(compute)
        for l in f.release_order:
            d = f.bwd_delay_s[l] * rng.uniform(0.9, 1.1)
            gr.gr_bench_spin(int(d * 1e9), max(1, sms - comm_sms), compute.cuda_stream)
            ctx2.gr_mark_ready_async(2 * l, ptrs[2 * l], compute.cuda_stream)
            ctx2.gr_mark_ready_async(2 * l + 1, ptrs[2 * l + 1], compute.cuda_stream)
        ev_bwd.record(compute)
        # cycle loop: one gr_step per tic while backward runs; once only the last group is
        # pending, one device-driven drain cycle (gr_step_drain) releases it the moment its
        # marks land, without waiting for the next tic or a host round trip
        nxt = time.perf_counter()
        left, complete = f.G, False
        while left > 1:
            rel, complete, _A, _ = ctx2.gr_step(bits=False)
            left -= len(rel)
            if complete:
                break
            nxt += cyc
            while time.perf_counter() < nxt:
                pass
        if not complete:
            ctx2.gr_step_drain()
        ctx2.gr_wait()
        ev_end.record(compute)
        torch.cuda.synchronize()
        if step >= 2:
            exposed.append(max(0.0, ev_bwd.elapsed_time(ev_end)))
            bwd.append(ev_start.elapsed_time(ev_bwd))
            survey.append(max_over_ranks(ev_start.elapsed_time(ev_end)) - max_over_ranks(bwd[-1]))
    ex_max = [max_over_ranks(x) for x in exposed]
    ex_mean_local = float(np.mean(exposed))
    ex_mean = ex_mean_local
    if N > 1:
        tt = torch.tensor([ex_mean_local], dtype=torch.float64, device=dev)
        dist.all_reduce(tt)
        ex_mean = float(tt.item()) / N
    out = {}
    # headline: SURVEY.md §8(d) cfg3's definition (max_r end of comm - max_r end of backward)
    out["exposed_comm_ms"] = round(max(0.0, float(np.mean(survey))), 4)
    out["exposed_comm"] = {"ms_per_step_max_over_ranks": round(float(np.mean(ex_max)), 4),
                           "ms_per_step_mean_over_ranks": round(ex_mean, 4),
                           "ms_per_step_survey_def": round(max(0.0, float(np.mean(survey))), 4),
                           "t_bwd_ms": round(float(np.mean(bwd)), 3),
                           "frac_of_bwd": round(max(0.0, float(np.mean(survey))) / float(np.mean(bwd)), 5),
                           "frac_of_bwd_max_over_ranks": round(float(np.mean(ex_max)) / float(np.mean(bwd)), 5),
                           "cycle_us": cycle_us, "comm_sms": comm_sms, "steps": len(exposed),
                           "compute": "gr_bench_spin per layer, d_l=2*OPS_l/(0.70*1401.8 TF/s) x U(0.9,1.1)",
                           "marks": "gr_mark_ready_async on the compute stream after each layer",
                           "cycles": "host tics while backward runs; the last group by gr_step_drain",
                           "survey_def": "max_r end of comm - max_r end of backward (SURVEY.md §8(d) cfg3)"}
    ctx2.gr_finalize()
    return out


def run_extras(args, ctx, grads, ptrs, tensor_order, f, N, rank, local, dev, compute, sms, barrier,
               max_over_ranks, gr):
    """cfg3 exposed comm (synthetic backward), cycle latency, NCCL baseline."""
    import numpy as np
    import torch
    import torch.distributed as dist

    out = exposed_comm(args, args.cycle_us, args.comm_sms, f, ptrs, N, rank, local, dev, compute, sms,
                       barrier, max_over_ranks, gr)

    # ---- NEXT-2 epilogue cost: the same step with the fused ||g||^2 / non-finite statistics ----
    batch = ctx.prepare_batch(tensor_order, [ptrs[t] for t in tensor_order])

    def step_stats():
        ctx.gr_mark_ready_prepared(batch)
        ctx.gr_step()
        ctx.gr_wait_async()

    ctx.gr_enable_grad_stats(True)
    for _ in range(3):
        step_stats()
    barrier()
    torch.cuda.synchronize()
    a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a0.record(compute)
    for _ in range(10):
        step_stats()
    a1.record(compute)
    torch.cuda.synchronize()
    out["ms_per_step_with_grad_stats"] = round(max_over_ranks(a0.elapsed_time(a1) / 10), 4)
    ctx.gr_enable_grad_stats(False)

    # ---- cfg3 per-group end-to-end bus bandwidth: one group released per cycle, group by group
    # (mark its tensors -> gr_step releases it -> its fused pack/reduce/unpack), timed with events
    # on the compute stream from before the marks to after gr_released_wait_async ----
    if N > 1:
        members = {}
        for t in tensor_order:
            members.setdefault(int(f.group_of[t]), []).append(t)
        gorder = list(dict.fromkeys(int(f.group_of[t]) for t in tensor_order))  # reverse-layer release
        per = {g: [] for g in gorder}
        pb_ = 2 if args.buffer == "f16" else 4
        for rep in range(6):
            evs = []
            barrier()
            torch.cuda.synchronize()
            for g in gorder:
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(compute)
                ids = members[g]
                ctx.gr_mark_ready_batch(ids, [ptrs[t] for t in ids])
                rel, _complete, _A, _ = ctx.gr_step(bits=False)
                assert rel == [g], (rel, g)
                ctx.gr_released_wait_async(compute.cuda_stream)
                e1.record(compute)
                evs.append((g, e0, e1))
            ctx.gr_wait()
            torch.cuda.synchronize()
            if rep >= 1:
                for g, e0, e1 in evs:
                    per[g].append(e0.elapsed_time(e1))
        rows = []
        for g in sorted(per):
            ms_g = max_over_ranks(statistics.median(per[g]))
            Sg = int(sum(int(f.numel[t]) for t in members[g])) * pb_
            rows.append({"group": g, "bytes": Sg, "ms": round(ms_g, 4),
                         "busbw_GBps": round(Sg * 2 * (N - 1) / N / (ms_g * 1e-3) / 1e9, 1)})
        out["per_group_e2e"] = {"groups": rows,
                                "what": "one group per cycle in reverse-layer order: mark its tensors -> gr_step -> "
                                        "fused pack/reduce/unpack; events on the compute stream around marks..."
                                        "gr_released_wait_async; median of 5 steps, max over ranks; busbw = "
                                        "S_g*2(N-1)/N/t (SURVEY.md §8(d) cfg3: >=720 GB/s target for g4/g5/g6)"}

    # ---- bitvector-only cycle latency (no tensor ready: pure coordination round) ----
    lat = []
    barrier()
    for i in range(300):
        t0 = time.perf_counter()
        ctx.gr_step()
        lat.append((time.perf_counter() - t0) * 1e6)
    # finish the (empty) step: mark everything so the context returns to a clean state
    for t in tensor_order:
        ctx.gr_mark_ready(t, ptrs[t])
    ctx.gr_step()
    ctx.gr_wait()
    lat = lat[50:]
    out["cycle_latency_us"] = {"p50": round(float(np.percentile(lat, 50)), 2),
                               "p99": round(float(np.percentile(lat, 99)), 2), "T": f.T,
                               "what": "host wall time of one gr_step with nothing released (launch + "
                                       "populate + NVLink AND + release + host hand-off)"}

    # ---- NCCL baseline on the same fused message (N > 1) ----
    if N > 1:
        E = int(f.numel.sum())
        dt = torch.float16 if args.buffer == "f16" else torch.float32
        fused = torch.empty(E, dtype=dt, device=dev)

        def nccl_step():
            torch.cat([g.view(-1) for g in grads], out=fused) if dt == torch.float32 else \
                fused.copy_(torch.cat([g.view(-1) for g in grads]))
            dist.all_reduce(fused, op=dist.ReduceOp.AVG)
            off = 0
            for g in grads:
                n = g.numel()
                g.copy_(fused[off:off + n])
                off += n

        for _ in range(3):
            nccl_step()
        barrier()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(5):
            nccl_step()
        b.record()
        torch.cuda.synchronize()
        ms_n = max_over_ranks(a.elapsed_time(b) / 5)
        a.record()
        for _ in range(5):
            dist.all_reduce(fused, op=dist.ReduceOp.AVG)
        b.record()
        torch.cuda.synchronize()
        ms_ar = max_over_ranks(a.elapsed_time(b) / 5)
        S = E * (2 if dt == torch.float16 else 4)
        out["nccl_baseline"] = {"step_ms": round(ms_n, 4),
                                "step_value_GBps": round(N * E * 4 / (ms_n * 1e-3) / 1e9, 3),
                                "allreduce_only_ms": round(ms_ar, 4),
                                "allreduce_busbw_GBps": round(S / (ms_ar * 1e-3) * 2 * (N - 1) / N / 1e9, 2),
                                "what": "torch.cat pack + NCCL all_reduce(AVG) + copy unpack on the same message"}
    return out


if __name__ == "__main__":
    main()
