# r02 call ff (4 GPUs): persistent armed kernel at real N>1 — armed multi-GPU parity, bench N=4/2,
# cfg4 cycle latency with armed cycles (T <= 1024, no skew, no baselines)
P=gpurun_out/r34
python -c "import __graft_entry__ as g; g.build()" > ${P}_build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "multi_gpu_armed or multi_gpu_step_drain" > ${P}_pytest_multi.log 2>&1; echo "multi rc $?"; tail -2 ${P}_pytest_multi.log
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 600 $TR --nproc-per-node 4 --master-port 29621 bench.py --gpus 4 > ${P}_bench_n4.log 2>&1; echo "bench n4 rc $?"; tail -1 ${P}_bench_n4.log | head -c 400; echo
timeout 600 $TR --nproc-per-node 2 --master-port 29622 bench.py --gpus 2 > ${P}_bench_n2.log 2>&1; echo "bench n2 rc $?"; tail -1 ${P}_bench_n2.log | head -c 400; echo
timeout 600 $TR --nproc-per-node 4 --master-port 29623 tools/bench_cfg4.py --no-baselines --tmax 1024 --skew-us 0 --cycles 5000 > ${P}_cfg4_n4_armed.jsonl 2>${P}_cfg4_n4.err; echo "cfg4 n4 rc $?"; cat ${P}_cfg4_n4_armed.jsonl
timeout 600 $TR --nproc-per-node 2 --master-port 29624 tools/bench_cfg4.py --no-baselines --tmax 1024 --skew-us 0 --cycles 5000 > ${P}_cfg4_n2_armed.jsonl 2>${P}_cfg4_n2.err; echo "cfg4 n2 rc $?"; cat ${P}_cfg4_n2_armed.jsonl
