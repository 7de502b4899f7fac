# r02 call c (4 GPUs): push-path parity on virtual ranks, NVLink counter calibration, real
# multi-process parity, bench N=2/4 pull vs push, cfg5 mid-size sweep pull vs push, 64 MiB trace.
P=gpurun_out/r3
python -c "import __graft_entry__ as g; g.build()" > ${P}_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_virtual.py -m gpu -x -q -k push > ${P}_pytest_push.log 2>&1; prc=$?; echo "push pytest rc $prc"
timeout 120 python tools/nvlink_counters.py > ${P}_nvl_cal.log 2>&1; echo "nvl cal rc $?"
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 400 $TR --nproc-per-node 4 --master-port 29511 bench.py --gpus 4 --steps 20 --warmup 5 > ${P}_bench_n4_pull.log 2>&1; echo "bench n4 pull rc $?"
timeout 400 $TR --nproc-per-node 2 --master-port 29512 bench.py --gpus 2 --steps 20 --warmup 5 > ${P}_bench_n2_pull.log 2>&1; echo "bench n2 pull rc $?"
if [ $prc -eq 0 ]; then
  GR_PUSH=1 timeout 300 $TR --nproc-per-node 4 --master-port 29513 bench.py --gpus 4 --steps 20 --warmup 5 --no-extras > ${P}_bench_n4_push.log 2>&1; echo "bench n4 push rc $?"
  GR_PUSH=1 timeout 300 $TR --nproc-per-node 2 --master-port 29514 bench.py --gpus 2 --steps 20 --warmup 5 --no-extras > ${P}_bench_n2_push.log 2>&1; echo "bench n2 push rc $?"
  bash tools/sweep_cfg5.sh 4 1024 1024 "GR_PUSH=0" "GR_PUSH=1" > ${P}_sw5_n4.txt 2>&1
  bash tools/sweep_cfg5.sh 2 1024 1024 "GR_PUSH=0" "GR_PUSH=1" > ${P}_sw5_n2.txt 2>&1
  for PU in 0 1; do
    GR_PUSH=$PU GR_TRACE=gpurun_out/tr64_push$PU GR_TRACE_MAX_CYCLES=8 timeout 200 $TR --nproc-per-node 4 --master-port 2952$PU tools/bench_cfg5.py --quick --min-kib 65536 --max-mib 64 --iters 5 > /dev/null 2>&1
    python tools/trace_summary.py gpurun_out/tr64_push$PU > ${P}_trace64_push$PU.txt 2>&1
  done
fi
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k multi_gpu > ${P}_pytest_multi.log 2>&1; echo "multi pytest rc $?"
