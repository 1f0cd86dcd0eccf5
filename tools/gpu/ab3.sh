for r in 1 2; do
echo "== default auto" >> gpurun_out/ab3.log; ENGINES=3 timeout 300 python tools/probe.py 512x256 256x1024 4096x1 >> gpurun_out/ab3.log 2>&1
echo "== default tma3 (5 CTAs)" >> gpurun_out/ab3.log; ENGINES=6 timeout 300 python tools/probe.py 512x256 256x1024 4096x1 >> gpurun_out/ab3.log 2>&1
echo "== tma3 6 CTAs" >> gpurun_out/ab3.log; W1MG_CUDA_SO=$PWD/paper_1810_00118_b200/lib/ab/libw1mg_cuda_lb5.so ENGINES=6 timeout 300 python tools/probe.py 512x256 256x1024 4096x1 >> gpurun_out/ab3.log 2>&1
done
true
