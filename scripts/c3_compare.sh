python scripts/c3_sweep.py
python bench.py --steps 5 --no-cpu-baseline --no-training --no-e2e > gpurun_out/b3.json 2>/dev/null; python -c "
import json; d=json.load(open('gpurun_out/b3.json'))['roofline_fine_sweep_c3']; print('bench leg', d['ms_per_sweep'], d['frac'], d['clocks'])"
python scripts/c3_sweep.py
