set -x
timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "graph or determinism or device_entry" 2>&1 | tail -3
timeout 300 python bench.py --no-cpu-baseline --no-c3-sweep --no-e2e > gpurun_out/bench_c2_graph.json 2>&1
timeout 300 python bench.py --no-cpu-baseline --no-c3-sweep --no-e2e --no-graphs > gpurun_out/bench_c2_eager.json 2>&1
ls gpurun_out
