# r02 call hh (4 GPUs): the final build's full multi-GPU parity (torchrun N=2/4) and cfg5 small
# messages at N=4 with the persistent armed kernel
P=gpurun_out/r36
python -c "import __graft_entry__ as g; g.build()" > ${P}_build.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -q -k multi_gpu > ${P}_pytest_multi.log 2>&1; echo "multi rc $?"; tail -2 ${P}_pytest_multi.log
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 600 $TR --nproc-per-node 4 --master-port 29631 tools/bench_cfg5.py --buffer f16 --max-mib 16 > ${P}_cfg5_n4_small.jsonl 2>${P}_cfg5_n4.err; echo "cfg5 rc $?"; cat ${P}_cfg5_n4_small.jsonl | cut -c1-300
