timeout 1200 python -m pytest tests/test_gpu_parity.py -q -x -k "n1 or errors or async or drain or multi_gpu_cfg1 or multi_gpu_edge" > gpurun_out/pt_bv.log 2>&1; tail -2 gpurun_out/pt_bv.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29901 tools/bench_cfg4.py --cycles 1000 --skew-us 0,10 --no-baselines > gpurun_out/cfg4_d.jsonl 2> gpurun_out/cfg4_d.err
grep '^{' gpurun_out/cfg4_d.jsonl
