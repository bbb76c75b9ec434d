# full round: gpu tests, default bench (C2), C3 bench, launch list, ncu captures of the top kernels
set -x
timeout 600 python -m pytest tests -m gpu -q 2>&1 | tail -3
timeout 600 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; tail -c 3000 gpurun_out/bench_default.json
timeout 300 python bench.py --config C3 --steps 3 --no-cpu-baseline --no-c3-sweep > gpurun_out/bench_c3.json 2>&1; tail -c 600 gpurun_out/bench_c3.json
timeout 300 python bench.py --config C4 --steps 3 --no-cpu-baseline --no-c3-sweep > gpurun_out/bench_c4.json 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_default.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-c3-sweep > /dev/null 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:"k_pass_res|k_streamed_pass|k_agg0" -s 40 -c 6 -o gpurun_out/prof_c3_k2 python scripts/prof_target.py c3 > /dev/null 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:"k_fine_sweep|k_pinn_chain|k_delta" -s 0 -c 6 -o gpurun_out/prof_c2 python scripts/prof_target.py c2 > /dev/null 2>&1
ls gpurun_out
