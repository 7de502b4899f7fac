# r02 call p (1 GPU): armed cycles — full GPU suite, cycle latency armed vs not, smoke, bench N=1
P=gpurun_out/r17
python -c "import __graft_entry__ as g; g.build()" > ${P}_build.log 2>&1
timeout 1800 python -m pytest tests -m gpu -x -q > ${P}_pytest.log 2>&1; echo "pytest rc $?"; tail -2 ${P}_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > ${P}_smoke.log 2>&1; echo "smoke rc $?"
for A in 1 0; do
  GR_ARM=$A timeout 120 python tools/bench_cycle.py --iters 3000 | sed "s/^/GR_ARM=$A /" >> ${P}_cycle.txt 2>&1
  GR_ARM=$A timeout 120 python tools/bench_cycle.py --iters 3000 --release | sed "s/^/GR_ARM=$A /" >> ${P}_cycle.txt 2>&1
done
GR_TRACE=gpurun_out/trc2 GR_TRACE_MAX_CYCLES=2000 timeout 120 python tools/bench_cycle.py --iters 1500 >> ${P}_cycle.txt 2>&1
python tools/trace_summary.py gpurun_out/trc2 2>&1 | head -4 >> ${P}_cycle.txt
cat ${P}_cycle.txt
timeout 600 python bench.py > ${P}_bench_n1.log 2>&1; echo "bench rc $?"
tail -1 ${P}_bench_n1.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['roofline']['frac'], d['cycle_latency_us'], d['ms_per_step_with_grad_stats'], d['e2e']['ms_per_step'])"
