P=gpurun_out/r26
python -c "import __graft_entry__ as g; g.build()" > ${P}_build.log 2>&1
timeout 1200 python tools/stress.py --minutes 15 --seed 1 > ${P}_stress.log 2>&1; echo "stress rc $?"
tail -3 ${P}_stress.log
