# A/B of two library builds on the kernel probe (same box, interleaved)
for r in 1 2; do
for so in paper_1810_00118_b200/lib/libw1mg_cuda.so paper_1810_00118_b200/lib/ab/libw1mg_cuda_lb5.so; do
  echo "== $so" >> gpurun_out/ab.log
  W1MG_CUDA_SO=$PWD/$so timeout 300 python tools/probe.py 4096x1 512x256 256x1024 128x1024 >> gpurun_out/ab.log 2>&1
done
done
true
