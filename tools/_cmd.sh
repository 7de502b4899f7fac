timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29667 bench.py --gpus 4 --exposed-sweep 250:16,100:16,1000:16,5000:16,250:8,250:32,250:148 > gpurun_out/cfg3_sweep4.jsonl 2> gpurun_out/cfg3_sweep4.err
grep cfg3 gpurun_out/cfg3_sweep4.jsonl | cut -c1-260
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29801 tools/bench_cfg5.py --buffer f32 --min-kib 64 --max-mib 1024 --iters 10 > gpurun_out/cfg5_n4_f32.jsonl 2> gpurun_out/cfg5_n4_f32.err
tail -3 gpurun_out/cfg5_n4_f32.jsonl | cut -c1-300
