#!/bin/bash
# ThreadSanitizer build of the host runtime + the plain-C race test (tests/c/race_mark_step.c).
# compute-sanitizer is closed on this pool (profiles/r02/compute_sanitizer_closed.txt), so the
# host side's threading contract is checked with TSAN instead. Usage (GPU box):
#   bash tools/build_tsan.sh && build/tsan/race_mark_step
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
OUT=$ROOT/build/tsan
mkdir -p "$OUT"
NVCC=${NVCC:-/usr/local/cuda/bin/nvcc}
ARCH="-gencode arch=compute_100a,code=sm_100a"
CS=$ROOT/paper_1909_11150_b200/csrc
$NVCC $ARCH -O1 -g -std=c++17 -shared -Xcompiler -fPIC,-fsanitize=thread -ltsan \
  -I "$ROOT/include" -I "$CS" -cudart shared "$CS"/*.cu "$CS"/*.cpp -o "$OUT/libgr_tsan.so" -lcuda
$NVCC $ARCH -O1 -g -Xcompiler -fsanitize=thread,-pthread -ltsan -I "$ROOT/include" \
  "$ROOT/tests/c/race_mark_step.c" -x cu -o "$OUT/race_mark_step" -L "$OUT" -lgr_tsan -Xlinker -rpath="$OUT" -cudart shared
echo "built $OUT/race_mark_step"
