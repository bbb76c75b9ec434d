set -x
for g in 10 25; do
PR_PINN_G50=$g timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "pinn_G_both or pinn_G_single or pipelined" 2>&1 | tail -2
PR_PINN_G50=$g timeout 300 python bench.py --pinn-width 50 --pinn-layers 10 --no-cpu-baseline --no-c3-sweep > gpurun_out/bench_c2_paper_net_g$g.json 2>&1
done
