# r02 call t (4 GPUs): final-code multi-process parity (real ranks, armed cycles) + training X1
P=gpurun_out/r22
python -c "import __graft_entry__ as g; g.build()" > ${P}_build.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -q -rs -k multi_gpu > ${P}_pytest_multi.log 2>&1; echo "multi rc $?"; tail -3 ${P}_pytest_multi.log
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
for N in 1 2 4; do
  for I in none ours ddp; do
    if [ $N -eq 1 ] && [ $I != none ]; then continue; fi
    timeout 600 $TR --nproc-per-node $N --master-port 2962$N tools/bench_train.py --impl $I --batch 8 2>/dev/null | tail -1 >> ${P}_train.jsonl
  done
done
cat ${P}_train.jsonl | cut -c1-400
