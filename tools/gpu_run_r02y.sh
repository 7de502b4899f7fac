# r02 call y (1 GPU): preloading armed kernel — armed tests, full suite, cycle latency, bench N=1
P=gpurun_out/r27
python -c "import __graft_entry__ as g; g.build()" > ${P}_build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q > ${P}_pytest_all.log 2>&1; echo "pytest all rc $?"; tail -2 ${P}_pytest_all.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > ${P}_smoke.log 2>&1; echo "smoke rc $?"
for A in 1 0; do GR_ARM=$A timeout 120 python tools/bench_cycle.py --iters 3000 | sed "s/^/GR_ARM=$A /"; done > ${P}_cycle.txt 2>&1
GR_TRACE=gpurun_out/trc6 GR_TRACE_MAX_CYCLES=2000 timeout 120 python tools/bench_cycle.py --iters 1500 >> ${P}_cycle.txt 2>&1
python tools/trace_summary.py gpurun_out/trc6 2>&1 | head -4 >> ${P}_cycle.txt
cat ${P}_cycle.txt
timeout 600 python bench.py > ${P}_bench_n1.log 2>&1; echo "bench rc $?"
tail -1 ${P}_bench_n1.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['roofline']['frac'], d['cycle_latency_us'], d['ms_per_step_with_grad_stats'], d['e2e']['ms_per_step'], d['gpu_launches'], d.get('armed_cycles'), d.get('armed_expired'))"
timeout 1000 python tools/stress.py --minutes 12 --seed 2 > ${P}_stress.log 2>&1; echo "stress rc $?"; tail -2 ${P}_stress.log
