set -x
timeout 600 python -m pytest tests/test_gpu_parity.py -q -k "persistent or theta or cn" 2>&1 | tail -4
timeout 300 python bench.py --config C3 --fine-theta 0.5 --steps 3 --no-cpu-baseline --no-c3-sweep --no-e2e > gpurun_out/bench_c3_cn2.json 2>&1
ls gpurun_out
