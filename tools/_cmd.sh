for n in 2 4; do
for suite in "edge --seeds 0:4" "cfg1 --seeds 0:10" "stats --seeds 0:2" "fcn --seeds 5:6 --buffers f16" "drain --seeds 0:4"; do
GR_RS_SPLIT=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29555 tests/mp_worker.py --suite $suite > gpurun_out/split_$n.log 2>&1; echo "N=$n $suite rc=$?"; grep "mp_worker suite" gpurun_out/split_$n.log
done; done
bash tools/sweep.sh 4 "GR_RS_SPLIT=0" "GR_RS_SPLIT=1" "GR_RS_SPLIT=0" "GR_RS_SPLIT=1" > gpurun_out/sw_split4.txt 2>&1; cat gpurun_out/sw_split4.txt
bash tools/sweep.sh 2 "GR_RS_SPLIT=0" "GR_RS_SPLIT=1" > gpurun_out/sw_split2.txt 2>&1; cat gpurun_out/sw_split2.txt
bash tools/sweep_cfg5.sh 4 4096 256 "GR_RS_SPLIT=0" "GR_RS_SPLIT=1" > gpurun_out/sw5_split4.txt 2>&1; cat gpurun_out/sw5_split4.txt
