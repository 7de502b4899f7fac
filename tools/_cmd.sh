timeout 1700 python -m pytest tests/test_gpu_parity.py -q -x -k "oversubscribed" -s > gpurun_out/pt_os.log 2>&1; tail -30 gpurun_out/pt_os.log
