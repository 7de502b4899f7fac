#!/bin/bash
# tools/sweep_cfg5.sh N MIN_KIB MAX_MIB "ENV1 ENV2" "ENV..." ... : cfg5 size sweep (library default
# algorithm only, no NCCL) once per env set; prints bytes -> us per env set.
N=$1; MINK=$2; MAXM=$3; shift 3
i=0
for envs in "$@"; do
  i=$((i+1))
  env $envs timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
     --master-port $((29800+i)) tools/bench_cfg5.py --quick --min-kib $MINK --max-mib $MAXM --iters 20 \
     > gpurun_out/sw5_$i.jsonl 2> gpurun_out/sw5_$i.err
  python - "$envs" gpurun_out/sw5_$i.jsonl <<'PY'
import json, sys
rows = []
for l in open(sys.argv[2]):
    try:
        d = json.loads(l)
    except Exception:
        continue
    if "bytes" in d:
        rows.append(f"{d['bytes'] >> 20}M:{d['default_us']:.1f}")
print(f"{sys.argv[1]:40s} " + " ".join(rows) if rows else f"{sys.argv[1]} FAILED")
PY
done
