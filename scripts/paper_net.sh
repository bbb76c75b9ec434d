# the paper's 10x50 PINN as the coarse propagator at C2: parity tests, bench lines
set -x
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "pinn or pipelined" 2>&1 | tail -3
for act in tanh; do
timeout 300 python bench.py --pinn-width 50 --pinn-layers 10 --no-cpu-baseline --no-c3-sweep > gpurun_out/bench_c2_paper_net.json 2> gpurun_out/bench_c2_paper_net.err
done
tail -c 600 gpurun_out/bench_c2_paper_net.json; tail -3 gpurun_out/bench_c2_paper_net.err
timeout 300 python bench.py --no-cpu-baseline --no-c3-sweep > gpurun_out/bench_c2_default.json 2>&1; tail -c 300 gpurun_out/bench_c2_default.json
