P=gpurun_out/r30
python -c "import __graft_entry__ as g; g.build()" > ${P}_build.log 2>&1
timeout 1300 python tools/stress.py --minutes 20 --seed 3 > ${P}_stress.log 2>&1; echo "stress rc $?"; tail -2 ${P}_stress.log
