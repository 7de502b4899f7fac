# r02 call h (4 GPUs): 64 MiB N=4 traces at the best chunk rule; doorbell latency probe
P=gpurun_out/r8
python -c "import __graft_entry__ as g; g.build()" > ${P}_build.log 2>&1
nvcc -gencode arch=compute_100a,code=sm_100a -O2 tools/doorbell_probe.cu -o build/doorbell_probe -lcuda > /dev/null 2>&1
timeout 120 build/doorbell_probe > ${P}_doorbell.txt 2>&1; echo "doorbell rc $?"
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
i=0
for ENVS in "GR_CHUNK_DIV=592" "GR_CHUNK_DIV=592 GR_LAG1=888 GR_LAG2=2368" "GR_CHUNK_DIV=592 GR_LAG1=222 GR_LAG2=592"; do
  i=$((i+1))
  env $ENVS GR_TRACE=gpurun_out/tr8_$i GR_TRACE_MAX_CYCLES=8 timeout 200 $TR --nproc-per-node 4 --master-port 2954$i tools/bench_cfg5.py --quick --min-kib 65536 --max-mib 64 --iters 5 > /dev/null 2>&1
  (echo "== $ENVS"; python tools/trace_summary.py gpurun_out/tr8_$i) > ${P}_trace64_$i.txt 2>&1
done
