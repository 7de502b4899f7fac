# r02 call k (4 GPUs): stage size x queue lags x sub-tile progress at N=4 (8-256 MiB) + fcn220m
P=gpurun_out/r11
python -c "import __graft_entry__ as g; g.build()" > ${P}_build.log 2>&1
bash tools/sweep_cfg5.sh 4 8192 256 "GR_NVLS=0" "GR_STAGES=2 GR_STAGE_KB=96" "GR_STAGES=3 GR_STAGE_KB=64" \
  "GR_STAGES=2 GR_STAGE_KB=96 GR_LAG1=0 GR_LAG2=148 GR_PUB_QUANTUM=16384" \
  "GR_LAG1=0 GR_LAG2=148 GR_PUB_QUANTUM=8192" "GR_LAG1=0 GR_LAG2=296 GR_PUB_QUANTUM=8192" \
  "GR_LAG1=74 GR_LAG2=296 GR_PUB_QUANTUM=8192" "GR_LAG1=148 GR_LAG2=444 GR_PUB_QUANTUM=8192" > ${P}_sweep_n4.txt 2>&1
cat ${P}_sweep_n4.txt
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
for ST in "GR_NVLS=0" "GR_STAGES=2 GR_STAGE_KB=96" "GR_STAGES=2 GR_STAGE_KB=96 GR_CHUNK_DIV=148" "GR_STAGES=3 GR_STAGE_KB=64"; do
  echo "== $ST" >> ${P}_bench.txt
  env $ST timeout 300 $TR --nproc-per-node 4 --master-port 29572 bench.py --gpus 4 --steps 20 --warmup 5 --no-extras 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('N=4', d['ms_per_step'], d['busbw_GBps'], d['roofline']['kernel_ms'])" >> ${P}_bench.txt 2>&1
  env $ST timeout 300 $TR --nproc-per-node 2 --master-port 29573 bench.py --gpus 2 --steps 20 --warmup 5 --no-extras 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('N=2', d['ms_per_step'], d['busbw_GBps'], d['roofline']['kernel_ms'])" >> ${P}_bench.txt 2>&1
done
cat ${P}_bench.txt
