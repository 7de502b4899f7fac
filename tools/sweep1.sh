#!/bin/bash
# tools/sweep1.sh "ENV..." ... : N=1 bench (no extras) once per env set
i=0
for envs in "$@"; do
  i=$((i+1))
  env $envs python bench.py --steps 50 --warmup 5 --no-extras > gpurun_out/sw1_$i.json 2> gpurun_out/sw1_$i.err
  python - "$envs" gpurun_out/sw1_$i.json <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[2]).read().strip().splitlines()[-1])
    print(f"{sys.argv[1]:40s} step {d['ms_per_step']:.4f} ms  kernel {d['roofline']['kernel_ms']:.4f} ms  frac {d['roofline']['frac']:.3f} launches/step {d['launches_per_step']}")
except Exception as e:
    print(sys.argv[1], "FAILED", e)
PY
done
