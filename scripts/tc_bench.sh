set -x
timeout 600 python bench.py --config C5 --pinn-width 256 --pinn-layers 8 --pinn-prec fp16tc --steps 2 --no-cpu-baseline --no-c3-sweep --no-e2e > gpurun_out/bench_c5_256x8_fp16tc.json 2>&1
timeout 600 python bench.py --config C5 --pinn-width 256 --pinn-layers 8 --pinn-prec bf16tc --steps 2 --no-cpu-baseline --no-c3-sweep --no-e2e > gpurun_out/bench_c5_256x8_bf16tc.json 2>&1
timeout 600 python bench.py --config C5 --pinn-width 64 --pinn-layers 4 --pinn-prec fp16tc --steps 3 --no-cpu-baseline --no-c3-sweep --no-e2e > gpurun_out/bench_c5_64x4_fp16tc.json 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_pinn_chain_tc -c 1 -o gpurun_out/prof_tc_256x8_split python scripts/prof_tc.py 256 8 1 > /dev/null 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_pinn_chain_tc -c 1 -o gpurun_out/prof_tc_256x8_bf16 python scripts/prof_tc.py 256 8 2 > /dev/null 2>&1
ls gpurun_out
