# bench A/B on one box: default engines vs the three-sweep engine everywhere
timeout 900 python bench.py --no-cpu > gpurun_out/bench_a.json 2> gpurun_out/bench_a.err
W1MG_SWEEP=tma3 timeout 900 python bench.py --no-cpu > gpurun_out/bench_b.json 2> gpurun_out/bench_b.err
timeout 900 python bench.py --no-cpu > gpurun_out/bench_a2.json 2> gpurun_out/bench_a2.err
true
