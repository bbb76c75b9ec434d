# K2 paired persistent pass (k_pass_res2) vs k_pass_res: parity, then C3 fine-sweep timing
set -x
timeout 400 python -m pytest tests/test_gpu_parity.py -q -x -k "streamed or c3_size or fine_single or portfolio or theta" 2>&1 | tail -2
for cfg in "1 2 2 2" "1 2 2 3" "1 1 4 2" "1 1 2 2" "0 2 2 2"; do set -- $cfg
PR_K2_PAIR=$1 PR_K2_SP=$2 PR_K2_H=$3 PR_K2_STAGES=$4 PR_PROBE_ONE=1 timeout 200 python scripts/l2_probe.py 2>&1 | head -1
done
