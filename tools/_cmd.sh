GR_TRACE=gpurun_out/trf GR_TRACE_MAX_CYCLES=6 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29911 bench.py --gpus 4 --steps 3 --warmup 3 --no-extras > gpurun_out/trf.log 2>&1
python tools/trace_summary.py gpurun_out/trf > gpurun_out/trf_sum.txt 2>&1; rm -f gpurun_out/trf.rank*.jsonl
for n in 2 4; do
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29777 tools/bench_train.py --batch 8"
timeout 300 $R --impl ours >> gpurun_out/trf_train.jsonl 2>>gpurun_out/trf_train.err
timeout 300 $R --impl ours --drain-tail 8 >> gpurun_out/trf_train.jsonl 2>>gpurun_out/trf_train.err
timeout 300 $R --impl ddp >> gpurun_out/trf_train.jsonl 2>>gpurun_out/trf_train.err
done
timeout 300 python tools/bench_train.py --impl none --batch 8 >> gpurun_out/trf_train.jsonl 2>>gpurun_out/trf_train.err
