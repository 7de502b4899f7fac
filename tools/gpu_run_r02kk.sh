# r02 call kk (1 GPU): the final .so — armed-cycle tests and the N=1 full-size parity
P=gpurun_out/r39
python -c "import __graft_entry__ as g; g.build()" > ${P}_build.log 2>&1
timeout 200 python -m pytest tests/test_gpu_parity.py -q -x -m gpu -k "armed or fcn220m_n1" > ${P}_pytest.log 2>&1; echo "pytest rc $?"; tail -1 ${P}_pytest.log
