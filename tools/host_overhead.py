"""Break down the fixed per-step host/device overhead of mark -> gr_step -> gr_wait
on a tiny message (design input). Run plain (N=1) or under torchrun (N>1)."""
import os, sys, time, statistics, json
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import paper_1909_11150_b200 as gr

rank = int(os.environ.get("RANK", "0")); N = int(os.environ.get("WORLD_SIZE", "1")); local = int(os.environ.get("LOCAL_RANK", "0"))
torch.cuda.set_device(local)
ag = None
if N > 1:
    import torch.distributed as dist
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    ag = gr.make_allgather(None, local)
g = torch.randn(256, device="cuda")
comp = torch.cuda.current_stream()
ctx = gr.Context(rank=rank, world_size=N, device=local, numel=[256], group_of=[0], compute_stream=comp.cuda_stream, allgather=ag)
batch = ctx.prepare_batch([0], [g.data_ptr()])
tm, ts, tw = [], [], []
for i in range(2000):
    t0 = time.perf_counter(); ctx.gr_mark_ready_prepared(batch)
    t1 = time.perf_counter(); ctx.gr_step()
    t2 = time.perf_counter(); ctx.gr_wait()
    t3 = time.perf_counter()
    if i >= 200:
        tm.append((t1 - t0) * 1e6); ts.append((t2 - t1) * 1e6); tw.append((t3 - t2) * 1e6)
st = ctx.stats()
cyc = st.cycles
out = {"rank": rank, "N": N, "mark_us": statistics.median(tm), "gr_step_us": statistics.median(ts), "gr_wait_us": statistics.median(tw),
       "lib_host_step_us": st.host_step_us / cyc, "lib_wait_handoff_us": st.host_wait_us / cyc,
       "bitvector_device_us": st.bitvector_device_us / cyc}
# raw launch + sync reference
s = torch.cuda.Stream()
x = torch.zeros(1, device="cuda")
lt = []
for i in range(500):
    t0 = time.perf_counter()
    with torch.cuda.stream(s):
        x.add_(1)
    s.synchronize()
    lt.append((time.perf_counter() - t0) * 1e6)
out["torch_launch_plus_sync_us"] = statistics.median(lt[100:])
print(json.dumps({k: round(v, 2) if isinstance(v, float) else v for k, v in out.items()}), flush=True)
