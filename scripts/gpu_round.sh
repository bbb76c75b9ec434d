set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
timeout 600 python -m pytest tests -m gpu -q 2>&1 | tail -15
timeout 300 python bench.py > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; cat gpurun_out/bench_c2.json; tail -5 gpurun_out/bench_c2.err
timeout 300 python bench.py --coarse ie --no-cpu-baseline > gpurun_out/bench_c2ie.json 2>&1; cat gpurun_out/bench_c2ie.json
timeout 300 python bench.py --config C4 --steps 3 --no-cpu-baseline > gpurun_out/bench_c4.json 2>&1; cat gpurun_out/bench_c4.json
timeout 600 python bench.py --config C3 --steps 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_c3.json 2>&1; cat gpurun_out/bench_c3.json
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file gpurun_out/launches_c2.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1; wc -l gpurun_out/launches_c2.csv
