set -x
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "tensor" 2>&1 | tail -25
ls gpurun_out
