# r02 call cc (1 GPU): ncu --set full of the N=1 step's kernels with the final build
P=gpurun_out/r31
python -c "import __graft_entry__ as g; g.build()" > ${P}_build.log 2>&1
GR_ARM=0 timeout 300 python bench.py --steps 3 --warmup 3 --no-extras > ${P}_plain.log 2>&1 && \
  GR_ARM=0 timeout 900 ncu --set full --clock-control none --import-source on -k regex:"local_kernel|bitvector_kernel" -s 6 -c 4 -o gpurun_out/r31_n1_full python bench.py --steps 3 --warmup 3 --no-extras > ${P}_ncu.log 2>&1; echo "ncu rc $?"
