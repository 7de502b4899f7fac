bash tools/sweep1.sh "GR_LC_SUB=2048" "GR_LC_SUB=1024" > gpurun_out/sw1_u2c.txt 2>&1; cat gpurun_out/sw1_u2c.txt
cp paper_1909_11150_b200/libgr.so /tmp/libgr_u2.so; cp gpurun_out/var/libgr_u1.so paper_1909_11150_b200/libgr.so
bash tools/sweep1.sh "GR_LC_SUB=2048" "GR_LC_SUB=4096" "GR_LC_SUB=1024" > gpurun_out/sw1_u1.txt 2>&1; cat gpurun_out/sw1_u1.txt
