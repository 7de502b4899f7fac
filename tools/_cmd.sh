timeout 300 python bench.py --steps 3 --warmup 3 --no-extras > gpurun_out/plain2.json 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"local_kernel|bitvector" -s 4 -c 4 -o gpurun_out/r01c_n1_full python bench.py --steps 3 --warmup 3 --no-extras > gpurun_out/ncu_f.log 2>&1
echo rc=$?
