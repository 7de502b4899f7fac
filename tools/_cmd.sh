timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29801 tools/bench_cfg5.py --tensors 16 --min-kib 64 --max-mib 1024 --iters 10 > gpurun_out/cfg5_n4_t16.jsonl 2> gpurun_out/cfg5_n4_t16.err
grep bytes gpurun_out/cfg5_n4_t16.jsonl | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print(d['bytes'], d['tensors'], round(d['default_us'],1), round(d['default_drain_us'],1), round(d['nccl_us'],1), round(d['default_drain_busbw'],1), round(d['nccl_busbw'],1))
"
