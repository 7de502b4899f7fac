# r02 call g (4 GPUs): queue-shape sweep at N=4 (chunk size x lags x progress quantum), 8-256 MiB
P=gpurun_out/r7
python -c "import __graft_entry__ as g; g.build()" > ${P}_build.log 2>&1
bash tools/sweep_cfg5.sh 4 8192 256 "GR_NVLS=0" "GR_CHUNK_DIV=592" "GR_CHUNK_DIV=1184" \
  "GR_CHUNK_DIV=592 GR_LAG1=296 GR_LAG2=740" "GR_CHUNK_DIV=1184 GR_LAG1=296 GR_LAG2=740" \
  "GR_CHUNK_DIV=1184 GR_LAG1=444 GR_LAG2=1036" "GR_CHUNK_DIV=2368 GR_LAG1=296 GR_LAG2=740" \
  "GR_CHUNK_DIV=592 GR_PUB_QUANTUM=8192" "GR_CHUNK_DIV=592 GR_PUB_QUANTUM=16384 GR_LAG1=296 GR_LAG2=592" \
  "GR_CHUNK_DIV=1184 GR_PUB_QUANTUM=8192 GR_LAG1=296 GR_LAG2=592" > ${P}_sweep_n4.txt 2>&1
cat ${P}_sweep_n4.txt
