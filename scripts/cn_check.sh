set -x
timeout 600 python -m pytest tests/test_gpu_parity.py -q -k "theta or cn" 2>&1 | tail -15
timeout 600 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
ls gpurun_out
