timeout 900 python bench.py --no-cpu --no-e2e > gpurun_out/bab_a.json 2> gpurun_out/bab_a.err
W1MG_CUDA_SO=$PWD/paper_1810_00118_b200/lib/ab/libw1mg_cuda_w2.so timeout 900 python bench.py --no-cpu --no-e2e > gpurun_out/bab_b.json 2> gpurun_out/bab_b.err
timeout 900 python bench.py --no-cpu --no-e2e > gpurun_out/bab_a2.json 2> gpurun_out/bab_a2.err
true
