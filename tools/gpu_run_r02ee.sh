# r02 call ee (1 GPU): armed-kernel ack race fix (ack one cycle ahead) — armed tests incl. "late",
# the N=1 parity file, cycle latency, a soak on the seed that found the race
P=gpurun_out/r33
python -c "import __graft_entry__ as g; g.build()" > ${P}_build.log 2>&1
timeout 300 python -m pytest tests -q -x -m gpu -k "armed or autograd" > ${P}_armed.log 2>&1; echo "armed rc $?"; tail -2 ${P}_armed.log
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -m gpu > ${P}_parity.log 2>&1; echo "parity rc $?"; tail -2 ${P}_parity.log
for A in 1 0; do
  GR_ARM=$A timeout 120 python tools/bench_cycle.py --iters 10000 > ${P}_cycle_arm$A.jsonl 2>&1; tail -1 ${P}_cycle_arm$A.jsonl
done
timeout 800 python tools/stress.py --minutes 10 --seed 11 > ${P}_stress.log 2>&1; echo "stress rc $?"; tail -1 ${P}_stress.log
