set -x
timeout 240 python -m pytest tests/test_gpu_parity.py -q -x -k "streamed or c3_size or fine_single or portfolio" 2>&1 | tail -2
for cfg in "2 2 2" "1 2 3" "2 1 2"; do set -- $cfg; PR_K2_SP=$1 PR_K2_H=$2 PR_K2_STAGES=$3 timeout 200 python bench.py --config C3 --steps 3 --no-cpu-baseline --no-e2e --no-c3-sweep > gpurun_out/bench_c3_v11_$1_$2_$3.json 2>&1; done
PR_K2_SP=2 PR_K2_H=2 PR_K2_STAGES=2 timeout 200 ncu --set full --clock-control none --import-source on -k regex:k_pass_res -s 20 -c 2 -o gpurun_out/prof_v11d python scripts/prof_target.py c3 > /dev/null 2>&1
ls gpurun_out
