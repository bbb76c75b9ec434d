# full round: gpu tests, smoke, default bench (C2), C3/C4 bench lines, launch list, ncu captures
set -x
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -3
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -1
timeout 600 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; tail -c 1500 gpurun_out/bench_default.json
timeout 300 python bench.py --config C3 --steps 3 --no-cpu-baseline --no-c3-sweep > gpurun_out/bench_c3.json 2>&1
timeout 300 python bench.py --config C4 --steps 3 --no-cpu-baseline --no-c3-sweep > gpurun_out/bench_c4.json 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_default.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-c3-sweep --no-graphs > /dev/null 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:"k_parareal_pipe" -c 1 -o gpurun_out/prof_c2_pipe python scripts/prof_target.py c2 > /dev/null 2>&1
ls gpurun_out
timeout 300 python bench.py --pinn-width 50 --pinn-layers 10 --no-cpu-baseline --no-c3-sweep > gpurun_out/bench_c2_paper_net.json 2>&1
timeout 300 python bench.py --config C3 --coarse ie --iters 3 --no-cpu-baseline --no-c3-sweep > gpurun_out/bench_c3_ie.json 2>&1
ls gpurun_out
