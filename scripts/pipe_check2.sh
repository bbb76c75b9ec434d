set -x
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "pipelined or graph" 2>&1 | tail -4
timeout 300 python bench.py --no-cpu-baseline --no-c3-sweep --no-e2e --pinn-width 50 --pinn-layers 10 > gpurun_out/bench_c2_paper.json 2>&1
timeout 300 python bench.py --no-cpu-baseline --no-c3-sweep --no-e2e > gpurun_out/bench_c2_def.json 2>&1
ls gpurun_out
