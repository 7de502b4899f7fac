# r02 call e (4 GPUs): progress-word pipeline — virtual-rank parity first, then N=4 / N=2 sweeps
P=gpurun_out/r5
python -c "import __graft_entry__ as g; g.build()" > ${P}_build.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_virtual.py tests/test_abi_conformance.py -m gpu -x -q > ${P}_pytest_virtual.log 2>&1; prc=$?; echo "virtual pytest rc $prc"
if [ $prc -ne 0 ]; then exit 1; fi
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > ${P}_smoke.log 2>&1; echo "smoke rc $?"
timeout 200 python tools/bench_virtual.py --n 2 > ${P}_bvirt.log 2>&1; echo "bvirt rc $?"
timeout 200 python tools/bench_virtual.py --n 4 >> ${P}_bvirt.log 2>&1
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
bash tools/sweep_cfg5.sh 4 1024 1024 "GR_PUSH=0" "GR_PUSH=0 GR_CHUNK_DIV=592" "GR_PUSH=1" > ${P}_sw5_n4.txt 2>&1
bash tools/sweep_cfg5.sh 2 1024 1024 "GR_PUSH=0" "GR_PUSH=0 GR_CHUNK_DIV=296" > ${P}_sw5_n2.txt 2>&1
GR_TRACE=gpurun_out/tr64p GR_TRACE_MAX_CYCLES=8 timeout 200 $TR --nproc-per-node 4 --master-port 29531 tools/bench_cfg5.py --quick --min-kib 65536 --max-mib 64 --iters 5 > /dev/null 2>&1
python tools/trace_summary.py gpurun_out/tr64p > ${P}_trace64.txt 2>&1
timeout 400 $TR --nproc-per-node 4 --master-port 29532 bench.py --gpus 4 --steps 20 --warmup 5 > ${P}_bench_n4.log 2>&1; echo "bench n4 rc $?"
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k multi_gpu > ${P}_pytest_multi.log 2>&1; echo "multi pytest rc $?"
