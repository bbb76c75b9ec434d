# round-2 GPU run 15 (session 4, generation grid barrier in the pipelined tail): GPU tests,
# smoke, default bench, paper-net line, launch list of the default bench, ncu --set full of the pipe
set -x
O=gpurun_out/r02p; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -25 > $O/pytest.txt; tail -3 $O/pytest.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1; tail -2 $O/smoke.txt
timeout 900 python bench.py > $O/bench_default.json 2> $O/bench_default.err; tail -c 300 $O/bench_default.err
timeout 300 python bench.py --pinn-width 50 --pinn-layers 10 --no-cpu-baseline --no-training --no-c3-sweep > $O/bench_c2_paper_net.json 2>/dev/null
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_default.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-c3-sweep --no-training --no-graphs > /dev/null 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:"k_parareal_pipe" -c 1 -o $O/prof_c2_pipe python scripts/prof_target.py c2 > /dev/null 2>&1
ls -la $O
