for b in 8 2; do
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29777 tools/bench_train.py --batch $b"
for args in "--drain-tail 1 --comm-ctas 32" "--drain-tail 1 --comm-ctas 148 --groups 4" "--drain-tail 8"; do
timeout 300 $R --impl ours $args >> gpurun_out/tr7.jsonl 2>>gpurun_out/tr7.err
done
timeout 300 $R --impl ddp >> gpurun_out/tr7.jsonl 2>>gpurun_out/tr7.err
timeout 300 $R --impl ddp_fp16 >> gpurun_out/tr7.jsonl 2>>gpurun_out/tr7.err
timeout 300 python tools/bench_train.py --impl none --batch $b >> gpurun_out/tr7.jsonl 2>>gpurun_out/tr7.err
done
