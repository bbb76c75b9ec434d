set -x
timeout 300 python -m pytest tests/test_gpu_parity.py -q -k "persistent or c3_size or streamed" 2>&1 | tail -2
timeout 300 python bench.py --config C3 --steps 3 --no-cpu-baseline --no-c3-sweep --no-e2e > gpurun_out/bench_c3_pf.json 2>&1
ls gpurun_out
