# r02 call d (4 GPUs): NVLink SM-scaling probe, NVLink counter calibration (nvidia-smi), bench N=2
# (pull, with counters) and N=4 (push), TSAN race test of the host runtime.
P=gpurun_out/r4
python -c "import __graft_entry__ as g; g.build()" > ${P}_build.log 2>&1
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tools/sm_scaling_probe.cu -o build/sm_scaling_probe > /dev/null 2>&1
timeout 300 build/sm_scaling_probe > ${P}_sm_scaling.txt 2>&1; echo "probe rc $?"
nvidia-smi nvlink -h > ${P}_nvsmi_nvlink_help.txt 2>&1
timeout 120 python tools/nvlink_counters.py > ${P}_nvl_cal.log 2>&1; echo "nvl cal rc $?"
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 400 $TR --nproc-per-node 2 --master-port 29512 bench.py --gpus 2 --steps 20 --warmup 5 > ${P}_bench_n2_pull.log 2>&1; echo "bench n2 pull rc $?"
GR_PUSH=1 timeout 300 $TR --nproc-per-node 4 --master-port 29513 bench.py --gpus 4 --steps 20 --warmup 5 --no-extras > ${P}_bench_n4_push.log 2>&1; echo "bench n4 push rc $?"
(bash tools/build_tsan.sh > ${P}_tsan_build.log 2>&1 && TSAN_OPTIONS="halt_on_error=0 second_deadlock_stack=1" timeout 600 build/tsan/race_mark_step > ${P}_tsan_run.log 2>&1); echo "tsan rc $?"
