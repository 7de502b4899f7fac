# r02 call u (4 GPUs): split PACK / dependent queues — parity on virtual ranks, then N=4/N=2 perf
P=gpurun_out/r23
python -c "import __graft_entry__ as g; g.build()" > ${P}_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_virtual.py -m gpu -x -q -k split_queue > ${P}_pytest_split.log 2>&1; prc=$?; echo "split pytest rc $prc"; tail -2 ${P}_pytest_split.log
if [ $prc -ne 0 ]; then exit 1; fi
bash tools/sweep_cfg5.sh 4 4096 512 "GR_QUEUE=0" "GR_QUEUE=1" "GR_QUEUE=1 GR_LAGD=74" "GR_QUEUE=1 GR_LAGD=444" "GR_QUEUE=1 GR_LAGD=888" > ${P}_sweep_n4.txt 2>&1
cat ${P}_sweep_n4.txt
bash tools/sweep_cfg5.sh 2 4096 512 "GR_QUEUE=0" "GR_QUEUE=1" > ${P}_sweep_n2.txt 2>&1
cat ${P}_sweep_n2.txt
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
for Q in 0 1; do
  for N in 4 2; do
    GR_QUEUE=$Q timeout 300 $TR --nproc-per-node $N --master-port 2963$N bench.py --gpus $N --steps 20 --warmup 5 --no-extras 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('Q=$Q N=$N', d['ms_per_step'], d['busbw_GBps'], d['roofline']['kernel_ms'])" >> ${P}_bench.txt 2>&1
  done
done
GR_QUEUE=1 timeout 200 python tools/bench_virtual.py --n 2 >> ${P}_bench.txt 2>&1
GR_QUEUE=1 timeout 200 python tools/bench_virtual.py --n 4 >> ${P}_bench.txt 2>&1
cat ${P}_bench.txt
