set -x
mkdir -p gpurun_out
W1MG_PDHG_RS=1 W1MG_RS2_NOCOOP=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:pdhg_rs2_kernel -s 1 -c 1 -o /tmp/prof_rs2 python tools/pdhg_probe.py 150 256 > gpurun_out/rs_ncu_rs2.log 2>&1
ncu -i /tmp/prof_rs2.ncu-rep --page raw --csv > gpurun_out/rs_ncu_rs2_raw.csv 2>/dev/null
ncu -i /tmp/prof_rs2.ncu-rep --page source --csv > gpurun_out/rs_ncu_rs2_src.csv 2>/dev/null
rm -f /tmp/prof_rs2.ncu-rep
true
