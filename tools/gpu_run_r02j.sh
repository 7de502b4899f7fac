# r02 call j (1 GPU): per-chunk overhead of the xfer kernel, HBM-bound on virtual ranks
P=gpurun_out/r10
python -c "import __graft_entry__ as g; g.build()" > ${P}_build.log 2>&1
for CE in 8192 16384 32768 65536 131072; do
  GR_CHUNK_ELEMS=$CE timeout 200 python tools/bench_virtual.py --n 2 --steps 5 | sed "s/^/chunk=$CE /" >> ${P}_chunks.txt 2>&1
  GR_CHUNK_ELEMS=$CE timeout 200 python tools/bench_virtual.py --n 4 --steps 5 | sed "s/^/chunk=$CE /" >> ${P}_chunks.txt 2>&1
done
for ST in "GR_STAGES=2 GR_STAGE_KB=96" "GR_STAGES=6 GR_STAGE_KB=32" "GR_STAGES=8 GR_STAGE_KB=24"; do
  env $ST timeout 200 python tools/bench_virtual.py --n 2 --steps 5 | sed "s/^/$ST /" >> ${P}_chunks.txt 2>&1
done
cat ${P}_chunks.txt
