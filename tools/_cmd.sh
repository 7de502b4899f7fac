bash tools/sweep.sh 4 "GR_LAG1=296 GR_LAG2=592" "GR_LAG1=444 GR_LAG2=888" "GR_LAG1=296 GR_LAG2=888" "GR_LAG1=444 GR_LAG2=1184" "GR_LAG1=592 GR_LAG2=1184" "GR_LAG1=444 GR_LAG2=888" "GR_LAG1=296 GR_LAG2=592" > gpurun_out/sw_lag4b.txt 2>&1
bash tools/sweep.sh 2 "GR_LAG1=296 GR_LAG2=592" "GR_LAG1=444 GR_LAG2=888" "GR_LAG1=296 GR_LAG2=888" "GR_LAG1=444 GR_LAG2=1184" "GR_LAG1=592 GR_LAG2=1184" "GR_LAG1=444 GR_LAG2=888" "GR_LAG1=296 GR_LAG2=592" > gpurun_out/sw_lag2b.txt 2>&1
bash tools/sweep_cfg5.sh 4 4096 256 "GR_LAG1=296 GR_LAG2=592" "GR_LAG1=444 GR_LAG2=888" "GR_LAG1=592 GR_LAG2=1184" > gpurun_out/sw5_lag4.txt 2>&1
cat gpurun_out/sw_lag4b.txt gpurun_out/sw_lag2b.txt gpurun_out/sw5_lag4.txt
