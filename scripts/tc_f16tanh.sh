set -x
timeout 180 python -m pytest tests/test_gpu_parity.py -q -k "tensor" 2>&1 | tail -1
for cfg in "256 8" "128 4" "64 8" "64 4"; do set -- $cfg
timeout 300 python bench.py --config C5 --pinn-width $1 --pinn-layers $2 --pinn-prec bf16tc --steps 2 --no-cpu-baseline --no-c3-sweep --no-e2e > gpurun_out/bench_c5_$1x$2_bf16tc_h2.json 2>&1
done
