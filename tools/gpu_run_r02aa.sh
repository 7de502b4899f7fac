# r02 call aa (4 GPUs): queue lags around the default with the final kernel (fine chunks, 2 x 96 KB)
P=gpurun_out/r29
python -c "import __graft_entry__ as g; g.build()" > ${P}_build.log 2>&1
bash tools/sweep_cfg5.sh 4 8192 512 "GR_NVLS=0" "GR_LAG1=296 GR_LAG2=888" "GR_LAG1=592 GR_LAG2=1184" "GR_LAG1=444 GR_LAG2=888" "GR_LAG1=444 GR_LAG2=1776" "GR_LAG1=222 GR_LAG2=1184" > ${P}_sweep_lags_n4.txt 2>&1
cat ${P}_sweep_lags_n4.txt
