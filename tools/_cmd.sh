timeout 300 python bench.py --steps 3 --warmup 3 --no-extras > gpurun_out/plain.json 2>&1 && \
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 1500 --csv --log-file gpurun_out/r01b_n1_launches.csv python bench.py --steps 3 --warmup 3 --no-extras > gpurun_out/ncu_l.log 2>&1
echo rc=$?
