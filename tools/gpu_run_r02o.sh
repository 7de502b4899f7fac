# r02 call o (4 GPUs): final evidence — full GPU suite on 4 GPUs, bench N=1/2/4 with extras,
# cfg4 (11 T x 3 skews x 1e4 cycles) at N=2/4, cfg5 (with NCCL) at N=2/4
P=gpurun_out/r16
python -c "import __graft_entry__ as g; g.build()" > ${P}_build.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q -rs > ${P}_pytest_all.log 2>&1; echo "pytest rc $?"; tail -3 ${P}_pytest_all.log
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 600 python bench.py > ${P}_bench_n1.log 2>&1; echo "bench n1 rc $?"
timeout 900 $TR --nproc-per-node 2 --master-port 29601 bench.py --gpus 2 > ${P}_bench_n2.log 2>&1; echo "bench n2 rc $?"
timeout 900 $TR --nproc-per-node 4 --master-port 29602 bench.py --gpus 4 > ${P}_bench_n4.log 2>&1; echo "bench n4 rc $?"
timeout 1500 $TR --nproc-per-node 4 --master-port 29603 tools/bench_cfg5.py --buffer f16 > ${P}_cfg5_n4_f16.jsonl 2>${P}_cfg5_n4.err; echo "cfg5 n4 rc $?"
timeout 1500 $TR --nproc-per-node 2 --master-port 29604 tools/bench_cfg5.py --buffer f16 > ${P}_cfg5_n2_f16.jsonl 2>${P}_cfg5_n2.err; echo "cfg5 n2 rc $?"
timeout 1500 $TR --nproc-per-node 4 --master-port 29605 tools/bench_cfg5.py --buffer f32 --min-kib 1024 > ${P}_cfg5_n4_f32.jsonl 2>${P}_cfg5_n4f32.err; echo "cfg5 n4 f32 rc $?"
timeout 1800 $TR --nproc-per-node 4 --master-port 29606 tools/bench_cfg4.py > ${P}_cfg4_n4.jsonl 2>${P}_cfg4_n4.err; echo "cfg4 n4 rc $?"
timeout 1800 $TR --nproc-per-node 2 --master-port 29607 tools/bench_cfg4.py > ${P}_cfg4_n2.jsonl 2>${P}_cfg4_n2.err; echo "cfg4 n2 rc $?"
