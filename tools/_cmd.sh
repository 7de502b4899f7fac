timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pt_final2.log 2>&1; tail -3 gpurun_out/pt_final2.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -1
timeout 600 python bench.py > gpurun_out/final_n1.json 2> gpurun_out/final_n1.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29668 bench.py --gpus 2 > gpurun_out/final_n2.json 2> gpurun_out/final_n2.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29667 bench.py --gpus 4 > gpurun_out/final_n4.json 2> gpurun_out/final_n4.err
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29669 bench.py --impl reference --gpus 4 --steps 2 --warmup 1 > gpurun_out/final_ref4.json 2> gpurun_out/final_ref4.err
