set -x
timeout 180 python -m pytest tests/test_gpu_parity.py -q -x -k "tensor" 2>&1 | tail -1
for d in 1 0; do PR_TC_DEEP=$d timeout 300 python bench.py --config C5 --pinn-width 256 --pinn-layers 8 --pinn-prec bf16tc --steps 2 --no-cpu-baseline --no-c3-sweep --no-e2e > gpurun_out/bench_c5_256x8_bf16_deep$d.json 2>&1; done
PR_TC_DEEP=1 timeout 300 python bench.py --config C5 --pinn-width 256 --pinn-layers 4 --pinn-prec bf16tc --steps 2 --no-cpu-baseline --no-c3-sweep --no-e2e > gpurun_out/bench_c5_256x4_bf16_deep1.json 2>&1
PR_TC_DEEP=0 timeout 300 python bench.py --config C5 --pinn-width 256 --pinn-layers 4 --pinn-prec bf16tc --steps 2 --no-cpu-baseline --no-c3-sweep --no-e2e > gpurun_out/bench_c5_256x4_bf16_deep0.json 2>&1
