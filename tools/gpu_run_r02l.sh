# r02 call l2 (1 GPU): lag1=0 stall on virtual ranks with the extended GR_DEBUG_DUMP; item parity
P=gpurun_out/r13
python -c "import __graft_entry__ as g; g.build()" > ${P}_build.log 2>&1
for cfg in "GR_LAG1=0 GR_LAG2=74 GR_ITEMS_PER_CTA=0" "GR_LAG1=0 GR_LAG2=74"; do
  tag=$(echo $cfg | tr ' =' '__')
  echo "== $cfg" >> ${P}_out.txt
  env $cfg GR_DEBUG_DUMP=gpurun_out/dbg2_$tag timeout 200 python tools/debug_lag0.py --n 4 --mib 16 >> ${P}_out.txt 2>&1
done
timeout 1200 python -m pytest tests/test_gpu_virtual.py tests/test_abi_conformance.py -m gpu -x -q > ${P}_pytest_virtual.log 2>&1; echo "virtual pytest rc $?"
timeout 200 python tools/bench_virtual.py --n 2 >> ${P}_bvirt.log 2>&1
GR_STAGES=2 GR_STAGE_KB=96 timeout 200 python tools/bench_virtual.py --n 2 >> ${P}_bvirt.log 2>&1
timeout 200 python tools/bench_virtual.py --n 4 >> ${P}_bvirt.log 2>&1
cat ${P}_out.txt ${P}_bvirt.log
