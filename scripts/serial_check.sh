set -x
timeout 300 python bench.py --config C3 --steps 3 --no-cpu-baseline --no-c3-sweep --no-e2e > gpurun_out/bench_c3_a.json 2>&1
PR_K2_PIPE=0 timeout 300 python bench.py --config C3 --steps 3 --no-cpu-baseline --no-c3-sweep --no-e2e > gpurun_out/bench_c3_b.json 2>&1
PR_K2_STAGES=4 timeout 300 python bench.py --config C3 --steps 3 --no-cpu-baseline --no-c3-sweep --no-e2e > gpurun_out/bench_c3_c.json 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:"k_fine_sweep|k_pinn_chain|k_delta" -s 0 -c 6 -o gpurun_out/prof_c2 python scripts/prof_target.py c2 > /dev/null 2>&1
ls gpurun_out
