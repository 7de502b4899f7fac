# r02 call dd (1 GPU): persistent armed bitvector kernel (data kernels wait on the cycle tag) —
# armed tests, the full 1-GPU suite, cycle latency armed/unarmed, bench; then ncu --set full (N=1)
P=gpurun_out/r32
python -c "import __graft_entry__ as g; g.build()" > ${P}_build.log 2>&1
timeout 300 python -m pytest tests -q -x -m gpu -k "armed or autograd" > ${P}_armed.log 2>&1; echo "armed rc $?"; tail -2 ${P}_armed.log
timeout 900 python -m pytest tests -q -x -m gpu > ${P}_pytest.log 2>&1; echo "pytest rc $?"; tail -2 ${P}_pytest.log
for A in 1 0; do
  GR_ARM=$A timeout 120 python tools/bench_cycle.py --iters 5000 > ${P}_cycle_arm$A.jsonl 2>&1; tail -1 ${P}_cycle_arm$A.jsonl
  GR_ARM=$A timeout 120 python tools/bench_cycle.py --iters 3000 --release > ${P}_cycle_rel_arm$A.jsonl 2>&1; tail -1 ${P}_cycle_rel_arm$A.jsonl
done
timeout 300 python bench.py > ${P}_bench.log 2>&1; echo "bench rc $?"; tail -1 ${P}_bench.log | head -c 700; echo
timeout 600 python tools/stress.py --minutes 4 --seed 11 > ${P}_stress.log 2>&1; echo "stress rc $?"; tail -1 ${P}_stress.log
GR_ARM=0 timeout 300 python bench.py --steps 3 --warmup 3 --no-extras > ${P}_plain.log 2>&1 && \
  GR_ARM=0 timeout 900 ncu --set full --clock-control none --import-source on -k regex:"local_kernel|bitvector_kernel" -s 6 -c 4 -o gpurun_out/r32_n1_full python bench.py --steps 3 --warmup 3 --no-extras > ${P}_ncu.log 2>&1; echo "ncu rc $?"
