set -x
mkdir -p gpurun_out
cap() { # name regex iters n
W1MG_PDHG_RS=3 timeout 600 ncu --set full --clock-control none --import-source on -k regex:$2 -s 1 -c 1 -o /tmp/prof_$1 python tools/pdhg_probe.py $3 $4 > gpurun_out/rs_ncu_$1.log 2>&1
ncu -i /tmp/prof_$1.ncu-rep --page raw --csv > gpurun_out/rs_ncu_$1_raw.csv 2>/dev/null
ncu -i /tmp/prof_$1.ncu-rep --page source --csv > gpurun_out/rs_ncu_$1_src.csv 2>/dev/null
rm -f /tmp/prof_$1.ncu-rep
}
cap pf513 pdhg_rspf_kernel 150 512
true
