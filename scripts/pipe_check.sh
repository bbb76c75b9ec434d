set -x
timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "pipelined or graph" 2>&1 | tail -15
timeout 300 python bench.py --no-cpu-baseline --no-c3-sweep > gpurun_out/bench_c2_pipe.json 2>&1
timeout 300 python bench.py --fine-theta 0.5 --no-cpu-baseline --no-c3-sweep > gpurun_out/bench_c2_cn_pipe.json 2>&1
timeout 600 python -m pytest tests -m gpu -q 2>&1 | tail -3
ls gpurun_out
