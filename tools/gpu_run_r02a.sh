set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r1_build.log 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q -rs > gpurun_out/r1_pytest.log 2>&1; echo "pytest rc $?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r1_smoke.log 2>&1; echo "smoke rc $?"
timeout 600 python bench.py > gpurun_out/r1_bench.log 2>&1; echo "bench rc $?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r1_launches.csv python bench.py --steps 2 --warmup 3 --no-extras > gpurun_out/r1_ncu.log 2>&1; echo "ncu rc $?"
