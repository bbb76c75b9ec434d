set -x
PR_K2_GFAC=1 timeout 400 python -m pytest tests/test_gpu_parity.py -q -x -k "streamed or c3_size or fine_single or portfolio or theta" 2>&1 | tail -2
for g in 0 1; do for cfg in "2 2 2" "2 2 3" "1 2 2" "2 1 3"; do set -- $cfg
PR_K2_GFAC=$g PR_K2_SP=$1 PR_K2_H=$2 PR_K2_STAGES=$3 PR_PROBE_ONE=1 timeout 200 python scripts/l2_probe.py 2>&1 | head -1 | sed "s/^/gfac=$g sp=$1 h=$2 nst=$3 /"
done; done
