timeout 600 python bench.py > gpurun_out/v_n1.json 2> gpurun_out/v_n1.err; tail -1 gpurun_out/v_n1.json | cut -c1-200
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29668 bench.py --gpus 2 > gpurun_out/v_n2.json 2> gpurun_out/v_n2.err; tail -1 gpurun_out/v_n2.json | cut -c1-200
