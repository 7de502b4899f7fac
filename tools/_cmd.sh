for n in 2 4; do
for suite in "edge --seeds 0:3" "fcn --seeds 7:8 --buffers f16" "stats --seeds 0:2"; do
GR_NVLS=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29555 tests/mp_worker.py --suite $suite > gpurun_out/nsplit_$n.log 2>&1; echo "N=$n $suite rc=$?"; grep "mp_worker suite" gpurun_out/nsplit_$n.log
done; done
bash tools/sweep.sh 4 "GR_NVLS=1 GR_NRS_SPLIT=0" "GR_NVLS=1 GR_NRS_SPLIT=1" "GR_NVLS=1 GR_NRS_SPLIT=0" "GR_NVLS=1 GR_NRS_SPLIT=1" > gpurun_out/sw_nsplit4.txt 2>&1; cat gpurun_out/sw_nsplit4.txt
