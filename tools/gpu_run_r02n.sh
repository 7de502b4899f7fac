# r02 call n (4 GPUs): coarse/fine chunking per message + 2x96 KB stages — parity, then perf
P=gpurun_out/r15
python -c "import __graft_entry__ as g; g.build()" > ${P}_build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q -k "virtual or conformance or multi_gpu_cfg1 or multi_gpu_edge" > ${P}_pytest.log 2>&1; prc=$?; echo "pytest rc $prc"
tail -3 ${P}_pytest.log
if [ $prc -ne 0 ]; then exit 1; fi
bash tools/sweep_cfg5.sh 4 1024 1024 "GR_NVLS=0" "GR_FINE_BELOW=0" > ${P}_sweep_n4.txt 2>&1
bash tools/sweep_cfg5.sh 2 1024 1024 "GR_NVLS=0" "GR_FINE_BELOW=0" > ${P}_sweep_n2.txt 2>&1
cat ${P}_sweep_n4.txt ${P}_sweep_n2.txt
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
for N in 4 2; do
  timeout 300 $TR --nproc-per-node $N --master-port 2959$N bench.py --gpus $N --steps 20 --warmup 5 --no-extras 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('N=$N', d['ms_per_step'], d['busbw_GBps'], d['roofline']['kernel_ms'])" >> ${P}_bench.txt 2>&1
done
timeout 200 python tools/bench_virtual.py --n 2 >> ${P}_bench.txt 2>&1
timeout 200 python tools/bench_virtual.py --n 4 >> ${P}_bench.txt 2>&1
cat ${P}_bench.txt
