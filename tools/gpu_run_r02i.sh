# r02 call i (4 GPUs): what NCCL uses at N=4 (algorithms forced), our NVLS at mid sizes with the
# N x 148 chunk rule, fcn220m bench at N=4 / N=2 with the new chunk rule
P=gpurun_out/r9
python -c "import __graft_entry__ as g; g.build()" > ${P}_build.log 2>&1
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
NCCL_DEBUG=INFO NCCL_DEBUG_SUBSYS=TUNING,INIT timeout 120 $TR --nproc-per-node 4 --master-port 29561 tools/nccl_algo_probe.py --sizes-mib 64 --iters 3 > ${P}_nccl_debug.log 2>&1
for A in default Ring Tree NVLS; do
  if [ $A = default ]; then E=""; else E="NCCL_ALGO=$A"; fi
  env $E timeout 120 $TR --nproc-per-node 4 --master-port 29562 tools/nccl_algo_probe.py >> ${P}_nccl_algos.jsonl 2>${P}_nccl_$A.err
done
bash tools/sweep_cfg5.sh 4 8192 256 "GR_NVLS=0" "GR_NVLS=1" > ${P}_sw5_nvls.txt 2>&1
timeout 400 $TR --nproc-per-node 4 --master-port 29563 bench.py --gpus 4 --steps 20 --warmup 5 --no-extras > ${P}_bench_n4.log 2>&1; echo "bench n4 rc $?"
timeout 400 $TR --nproc-per-node 2 --master-port 29564 bench.py --gpus 2 --steps 20 --warmup 5 --no-extras > ${P}_bench_n2.log 2>&1; echo "bench n2 rc $?"
GR_CHUNK_DIV=148 timeout 400 $TR --nproc-per-node 2 --master-port 29565 bench.py --gpus 2 --steps 20 --warmup 5 --no-extras > ${P}_bench_n2_div148.log 2>&1; echo "bench n2 div148 rc $?"
