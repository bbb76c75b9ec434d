# C2 variants: the paper's CN fine propagator with PINN and numerical coarse G
set -x
timeout 300 python bench.py --fine-theta 0.5 --no-cpu-baseline --no-c3-sweep > gpurun_out/bench_c2_cn_pinn.json 2>&1
timeout 300 python bench.py --fine-theta 0.5 --coarse ie --no-cpu-baseline --no-c3-sweep > gpurun_out/bench_c2_cn_ie1.json 2>&1
timeout 300 python bench.py --fine-theta 0.5 --coarse ie --coarse-steps 50 --no-cpu-baseline --no-c3-sweep > gpurun_out/bench_c2_cn_ie50.json 2>&1
timeout 300 python bench.py --coarse ie --coarse-steps 50 --no-cpu-baseline --no-c3-sweep > gpurun_out/bench_c2_ie50.json 2>&1
timeout 300 python bench.py --config C1 --no-cpu-baseline --no-c3-sweep > gpurun_out/bench_c1.json 2>&1
