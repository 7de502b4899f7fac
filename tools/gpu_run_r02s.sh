# r02 call s (4 GPUs): graded fine chunks sweep; final bench N=2/4 and cfg5/cfg4 at N=4 with armed cycles
P=gpurun_out/r21
python -c "import __graft_entry__ as g; g.build()" > ${P}_build.log 2>&1
bash tools/sweep_cfg5.sh 4 4096 256 "GR_NVLS=0" "GR_FINE_HEAD=296" "GR_FINE_HEAD=444" "GR_FINE_HEAD=888" > ${P}_sweep_head_n4.txt 2>&1
cat ${P}_sweep_head_n4.txt
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 900 $TR --nproc-per-node 4 --master-port 29611 bench.py --gpus 4 > ${P}_bench_n4.log 2>&1; echo "bench n4 rc $?"
timeout 900 $TR --nproc-per-node 2 --master-port 29612 bench.py --gpus 2 > ${P}_bench_n2.log 2>&1; echo "bench n2 rc $?"
timeout 1500 $TR --nproc-per-node 4 --master-port 29613 tools/bench_cfg5.py --buffer f16 > ${P}_cfg5_n4_f16.jsonl 2>${P}_cfg5_n4.err; echo "cfg5 n4 rc $?"
timeout 1800 $TR --nproc-per-node 4 --master-port 29614 tools/bench_cfg4.py > ${P}_cfg4_n4.jsonl 2>${P}_cfg4_n4.err; echo "cfg4 n4 rc $?"
