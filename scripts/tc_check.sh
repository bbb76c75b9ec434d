set -x
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "tensor" 2>&1 | tail -4
timeout 900 python scripts/pinn_width.py 2>&1 | tail -9
ls gpurun_out
