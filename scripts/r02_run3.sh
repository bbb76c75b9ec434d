# round-2 GPU run 3: full GPU tests, smoke, default bench (with the training leg), reference arm
set -x
mkdir -p gpurun_out/r02c
timeout 1200 python -m pytest tests -m gpu -q 2>&1 | tail -25 > gpurun_out/r02c/pytest.txt; tail -3 gpurun_out/r02c/pytest.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02c/smoke.txt 2>&1; tail -2 gpurun_out/r02c/smoke.txt
timeout 900 python bench.py > gpurun_out/r02c/bench_default.json 2> gpurun_out/r02c/bench_default.err; tail -c 300 gpurun_out/r02c/bench_default.err
timeout 600 python bench.py --config C5 --pinn-width 256 --pinn-layers 8 --pinn-prec fp16tc --steps 3 --no-cpu-baseline --no-training --no-c3-sweep > gpurun_out/r02c/bench_c5_256x8.json 2>/dev/null
timeout 600 python bench.py --config C3 --steps 3 --no-cpu-baseline --no-training --no-c3-sweep > gpurun_out/r02c/bench_c3.json 2>/dev/null
ls -la gpurun_out/r02c
