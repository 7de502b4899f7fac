# r02 call gg (1 GPU): final validation of the round's last build — the driver's round-end legs
# (full pytest -m gpu, smoke, bench N=1, reference arm) and the ncu launch list of the N=1 step
P=gpurun_out/r35
python -c "import __graft_entry__ as g; g.build()" > ${P}_build.log 2>&1
timeout 1200 python -m pytest tests -q -m gpu > ${P}_pytest.log 2>&1; echo "pytest rc $?"; tail -2 ${P}_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > ${P}_smoke.log 2>&1; echo "smoke rc $?"; tail -1 ${P}_smoke.log
timeout 300 python bench.py > ${P}_bench.log 2>&1; echo "bench rc $?"; tail -1 ${P}_bench.log | head -c 300; echo
timeout 300 python bench.py --impl reference > ${P}_ref.log 2>&1; echo "ref rc $?"; tail -1 ${P}_ref.log | head -c 300; echo
timeout 300 python bench.py --steps 2 --warmup 3 --no-extras > ${P}_plain.log 2>&1 && \
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file ${P}_launches_n1.csv python bench.py --steps 2 --warmup 3 --no-extras > ${P}_ncu.log 2>&1; echo "ncu rc $?"
