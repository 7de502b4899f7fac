# r02 call f (1 GPU): coordination-latency breakdown, launch costs, ncu launch list (N=1 bench)
# and one ncu --set full capture of the virtual-rank xfer kernel (pack / RS / AG HBM traffic).
P=gpurun_out/r6
python -c "import __graft_entry__ as g; g.build()" > ${P}_build.log 2>&1
nvcc -gencode arch=compute_100a,code=sm_100a -O2 tools/api_cost.cu -o build/api_cost > /dev/null 2>&1 && timeout 60 build/api_cost > ${P}_api_cost.txt 2>&1
timeout 120 python tools/bench_cycle.py --iters 3000 > ${P}_cycle.txt 2>&1
GR_TRACE=gpurun_out/trc1 GR_TRACE_MAX_CYCLES=2000 timeout 120 python tools/bench_cycle.py --iters 1500 >> ${P}_cycle.txt 2>&1
python tools/trace_summary.py gpurun_out/trc1 2>&1 | head -8 >> ${P}_cycle.txt
timeout 120 python tools/bench_cycle.py --virtual 4 --iters 2000 >> ${P}_cycle.txt 2>&1
timeout 120 python tools/bench_cycle.py --release --iters 2000 >> ${P}_cycle.txt 2>&1
timeout 300 python bench.py --steps 2 --warmup 3 --no-extras > ${P}_b_plain.log 2>&1 && \
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"local_kernel|bitvector_kernel" -c 40 --csv --log-file ${P}_launches_n1.csv python bench.py --steps 2 --warmup 3 --no-extras > ${P}_ncu1.log 2>&1; echo "ncu1 rc $?"
timeout 300 python tools/bench_virtual.py --n 2 --steps 2 --warmup 1 > ${P}_bv_plain.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:xfer_kernel_v -s 1 -c 1 -o gpurun_out/r6_xfer_v2 python tools/bench_virtual.py --n 2 --steps 2 --warmup 1 > ${P}_ncu2.log 2>&1; echo "ncu2 rc $?"
