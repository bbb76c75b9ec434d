set -x
timeout 240 python -m pytest tests/test_gpu_parity.py -q -x -k "streamed or c3_size or portfolio_instances or fine_single" 2>&1 | tail -4
for S in 1 2 4; do PR_K2_S=$S timeout 200 python bench.py --config C3 --steps 3 --no-cpu-baseline --no-e2e --no-c3-sweep > gpurun_out/bench_c3_S$S.json 2>&1; done
timeout 400 python -m pytest tests -m gpu -q 2>&1 | tail -3
for S in 2 4; do PR_K2_S=$S timeout 200 ncu --set full --clock-control none --import-source on -k regex:k_streamed_pass -s 20 -c 2 -o gpurun_out/prof_k2_S$S python scripts/prof_target.py c3 > /dev/null 2>&1; done
ls gpurun_out
