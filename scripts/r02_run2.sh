# round-2 GPU run 2: full GPU tests, smoke, default bench, ncu launch list of the bench command,
# ncu --set full captures of the dominant kernels (traffic for bench's roofline), training kernel
set -x
mkdir -p gpurun_out/r02b
timeout 1200 python -m pytest tests -m gpu -q 2>&1 | tail -25 > gpurun_out/r02b/pytest.txt; tail -3 gpurun_out/r02b/pytest.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02b/smoke.txt 2>&1; tail -2 gpurun_out/r02b/smoke.txt
timeout 900 python bench.py > gpurun_out/r02b/bench_default.json 2> gpurun_out/r02b/bench_default.err; tail -c 400 gpurun_out/r02b/bench_default.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r02b/bench_reference.json 2>/dev/null
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02b/launches_default.csv python bench.py --steps 2 --warmup 1 --no-c3-sweep --no-training --no-cpu-baseline > gpurun_out/r02b/launches_bench.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_parareal_pipe -c 1 -o gpurun_out/r02b/prof_pipe_c2 python scripts/prof_target.py c2 > gpurun_out/r02b/prof_pipe.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_pass_res2 -s 4 -c 2 -o gpurun_out/r02b/prof_k2res2 python scripts/prof_target.py c3 > gpurun_out/r02b/prof_k2.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_train_grad -s 30 -c 1 -o gpurun_out/r02b/prof_train python scripts/train_time.py > gpurun_out/r02b/prof_train.log 2>&1
ls -la gpurun_out/r02b
