set -x
timeout 300 python bench.py --fine-theta 0.5 --no-cpu-baseline --no-c3-sweep > gpurun_out/bench_c2_cn.json 2>&1
timeout 300 python bench.py --config C3 --fine-theta 0.5 --steps 3 --no-cpu-baseline --no-c3-sweep --no-e2e > gpurun_out/bench_c3_cn.json 2>&1
timeout 300 python bench.py --config C4 --fine-theta 0.5 --steps 3 --no-cpu-baseline --no-c3-sweep --no-e2e > gpurun_out/bench_c4_cn.json 2>&1
ls gpurun_out
