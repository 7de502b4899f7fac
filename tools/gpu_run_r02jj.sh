# r02 call jj (1 GPU): the round's last build — full pytest -m gpu and smoke (the driver's legs)
P=gpurun_out/r38
python -c "import __graft_entry__ as g; g.build()" > ${P}_build.log 2>&1
timeout 540 python -m pytest tests -q -m gpu -x > ${P}_pytest.log 2>&1; echo "pytest rc $?"; tail -2 ${P}_pytest.log
timeout 120 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > ${P}_smoke.log 2>&1; echo "smoke rc $?"; tail -1 ${P}_smoke.log
