set -x
timeout 240 python -m pytest tests/test_gpu_parity.py -q -x -k "streamed or c3_size or portfolio_instances or fine_single" 2>&1 | tail -4
timeout 400 python -m pytest tests -m gpu -q 2>&1 | tail -5
timeout 300 python bench.py --config C3 --steps 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_c3.json 2>&1; cut -c1-200 gpurun_out/bench_c3.json
timeout 200 ncu --set full --clock-control none --import-source on -k regex:k_streamed_pass -s 20 -c 2 -o gpurun_out/prof_streamed13 python scripts/prof_target.py c3 > /dev/null 2>&1
ls gpurun_out
