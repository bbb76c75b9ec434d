set -x
timeout 180 python -m pytest tests/test_gpu_parity.py -q -x -k "tensor" 2>&1 | tail -3
timeout 300 python bench.py --config C5 --pinn-width 256 --pinn-layers 8 --pinn-prec bf16tc --steps 2 --no-cpu-baseline --no-c3-sweep --no-e2e > gpurun_out/bench_c5_256x8_bf16tc_pp.json 2>&1
PR_TC_PINGPONG=0 timeout 300 python bench.py --config C5 --pinn-width 256 --pinn-layers 8 --pinn-prec bf16tc --steps 2 --no-cpu-baseline --no-c3-sweep --no-e2e > gpurun_out/bench_c5_256x8_bf16tc_old.json 2>&1
timeout 300 python bench.py --config C5 --pinn-width 128 --pinn-layers 4 --pinn-prec bf16tc --steps 2 --no-cpu-baseline --no-c3-sweep --no-e2e > gpurun_out/bench_c5_128x4_bf16tc_pp.json 2>&1
PR_TC_PINGPONG=0 timeout 300 python bench.py --config C5 --pinn-width 128 --pinn-layers 4 --pinn-prec bf16tc --steps 2 --no-cpu-baseline --no-c3-sweep --no-e2e > gpurun_out/bench_c5_128x4_bf16tc_old.json 2>&1
