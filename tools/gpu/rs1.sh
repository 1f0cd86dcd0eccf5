set -x
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_pdhg.py -x -q -p no:cacheprovider -k "fixed_iterations or config3 or converged" > gpurun_out/rs1_tests.log 2>&1; echo rc $? >> gpurun_out/rs1_tests.log
for rs in 0 3 2; do
W1MG_PDHG_RS=$rs W1MG_PERSIST_STAMPS=1 timeout 300 python tools/pdhg_probe.py 200 32 64 128 256 512 > gpurun_out/rs1_probe_rs$rs.log 2>&1
done
W1MG_PDHG_RS=1 timeout 300 python tools/configs.py 3 > gpurun_out/rs1_cfg3.log 2>&1
true
