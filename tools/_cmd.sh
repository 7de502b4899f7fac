bash tools/sweep.sh 4 "GR_NVLS=0" "GR_NVLS=1" "GR_NVLS=1 GR_CHUNK_DIV=148" > gpurun_out/sw_nvls3.txt 2>&1
