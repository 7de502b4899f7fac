# r02 call z (4 GPUs): final-code N=2/4 bench lines, multi-process parity, cfg5 at N=2 and N=4
P=gpurun_out/r28
python -c "import __graft_entry__ as g; g.build()" > ${P}_build.log 2>&1
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 900 $TR --nproc-per-node 4 --master-port 29641 bench.py --gpus 4 > ${P}_bench_n4.log 2>&1; echo "bench n4 rc $?"
timeout 900 $TR --nproc-per-node 2 --master-port 29642 bench.py --gpus 2 > ${P}_bench_n2.log 2>&1; echo "bench n2 rc $?"
timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -q -k multi_gpu > ${P}_pytest_multi.log 2>&1; echo "multi rc $?"; tail -2 ${P}_pytest_multi.log
timeout 1500 $TR --nproc-per-node 2 --master-port 29643 tools/bench_cfg5.py --buffer f16 > ${P}_cfg5_n2_f16.jsonl 2>${P}_cfg5_n2.err; echo "cfg5 n2 rc $?"
timeout 1500 $TR --nproc-per-node 4 --master-port 29644 tools/bench_cfg5.py --buffer f16 > ${P}_cfg5_n4_f16.jsonl 2>${P}_cfg5_n4.err; echo "cfg5 n4 rc $?"
