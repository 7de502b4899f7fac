for d in 296 148; do
GR_CHUNK_DIV=$d timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29667 bench.py --gpus 4 > gpurun_out/bench_n4_d$d.json 2> gpurun_out/bench_n4_d$d.err
GR_CHUNK_DIV=$d timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29668 bench.py --gpus 2 > gpurun_out/bench_n2_d$d.json 2> gpurun_out/bench_n2_d$d.err
done
