# r02 call ii (2 GPUs): persistent armed kernel restricted to N=1 (one cycle per armed kernel at
# N>1, event-ordered data kernel) — the multi-GPU suites that timed out in r36, and bench N=2
P=gpurun_out/r37
python -c "import __graft_entry__ as g; g.build()" > ${P}_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "multi_gpu_fcn220m or multi_gpu_armed or multi_gpu_nvls" > ${P}_pytest_multi.log 2>&1; echo "multi rc $?"; tail -2 ${P}_pytest_multi.log
timeout 600 python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --nproc-per-node 2 --master-port 29641 bench.py --gpus 2 > ${P}_bench_n2.log 2>&1; echo "bench n2 rc $?"; tail -1 ${P}_bench_n2.log | head -c 300; echo
