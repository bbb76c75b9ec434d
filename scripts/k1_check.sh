set -x
timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "fine_single or serial_fine or theta or pipelined" 2>&1 | tail -2
for wv in 0 1; do PR_K1_WIDE=$wv timeout 300 python bench.py --no-cpu-baseline --no-c3-sweep --no-e2e > gpurun_out/bench_k1_$wv.json 2>&1; done
python - <<'PY'
import os, sys, json
sys.path.insert(0, '.')
from paper_2303_03848_b200 import parareal, synth
for wv in ("0", "1"):
    os.environ["PR_K1_WIDE"] = wv
PY
ls gpurun_out
