P=gpurun_out/r25
python -c "import __graft_entry__ as g; g.build()" > ${P}_build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "armed" > ${P}_pytest.log 2>&1; echo "pytest rc $?"; tail -2 ${P}_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > ${P}_smoke.log 2>&1; echo "smoke rc $?"
