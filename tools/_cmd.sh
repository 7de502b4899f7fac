timeout 1200 python -m pytest tests/test_gpu_parity.py -q -x -k "multi_gpu_cfg1 or multi_gpu_edge or multi_gpu_fcn or multi_gpu_stats or multi_gpu_grad or multi_gpu_step" > gpurun_out/pt_push.log 2>&1; tail -3 gpurun_out/pt_push.log
bash tools/sweep.sh 4 "GR_PUSH=0" "GR_PUSH=1" "GR_PUSH=0" "GR_PUSH=1" > gpurun_out/sw_push4.txt 2>&1
bash tools/sweep.sh 2 "GR_PUSH=0" "GR_PUSH=1" "GR_PUSH=0" "GR_PUSH=1" > gpurun_out/sw_push2.txt 2>&1
cat gpurun_out/sw_push4.txt gpurun_out/sw_push2.txt
