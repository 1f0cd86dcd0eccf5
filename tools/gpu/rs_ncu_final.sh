set -x
mkdir -p gpurun_out
cap() { # name regex iters n extra-env
env $5 timeout 600 ncu --set full --clock-control none --import-source on -k regex:$2 -s 1 -c 1 -o /tmp/prof_$1 python tools/pdhg_probe.py $3 $4 > gpurun_out/ncuf_$1.log 2>&1
ncu -i /tmp/prof_$1.ncu-rep --page raw --csv > gpurun_out/ncuf_$1_raw.csv 2>/dev/null
rm -f /tmp/prof_$1.ncu-rep
}
cap 129 pdhg_rs_kernel 300 128 W1MG_PDHG_RS=1
cap 257 pdhg_rs2_kernel 150 256 "W1MG_PDHG_RS=1 W1MG_RS2_NOCOOP=1"
cap 513 pdhg_rspf_kernel 150 512 W1MG_PDHG_RS=1
true
