for g in "" "--no-graphs"; do timeout 300 python bench.py --no-cpu-baseline --no-c3-sweep --no-e2e $g > gpurun_out/bench_ge$g.json 2>&1; done
ls gpurun_out
