timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pt_final.log 2>&1; tail -3 gpurun_out/pt_final.log
timeout 600 python bench.py > gpurun_out/bench_n1.json 2> gpurun_out/bench_n1.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29668 bench.py --gpus 2 > gpurun_out/bench_n2.json 2> gpurun_out/bench_n2.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29667 bench.py --gpus 4 > gpurun_out/bench_n4.json 2> gpurun_out/bench_n4.err
