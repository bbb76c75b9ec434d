set -x
timeout 600 python -m pytest tests -m gpu -q 2>&1 | tail -8
timeout 600 python bench.py --config C3 --steps 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_c3.json 2>&1; cat gpurun_out/bench_c3.json | cut -c1-300
timeout 300 python bench.py > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; cat gpurun_out/bench_c2.json | cut -c1-300
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_streamed_pass -s 20 -c 2 -o gpurun_out/prof_streamed7 python scripts/prof_target.py c3 > /dev/null 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_pinn_chain -s 1 -c 1 -o gpurun_out/prof_pinn7_c2 python scripts/prof_target.py c2 > /dev/null 2>&1
ls gpurun_out
