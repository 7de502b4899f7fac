#!/bin/bash
# tools/sweep.sh N "ENV1 ENV2" "ENV..." ... : run the N-GPU bench (no extras) once per env set
N=$1; shift
i=0
for envs in "$@"; do
  i=$((i+1))
  env $envs timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
     --master-port $((29700+i)) bench.py --gpus $N --steps 10 --warmup 3 --no-extras > gpurun_out/sweep_$i.json 2> gpurun_out/sweep_$i.err
  python - "$envs" gpurun_out/sweep_$i.json <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[2]).read().strip().splitlines()[-1])
    print(f"{sys.argv[1]:50s} step {d['ms_per_step']:.4f} ms  kernel {d['roofline']['kernel_ms']:.4f} ms  frac {d['roofline']['frac']:.3f}  busbw {d['busbw_GBps']}  algo {d['config']['algo']}")
except Exception as e:
    print(sys.argv[1], "FAILED", e)
PY
done
