# variation of the C3 fine-sweep timing: the bench leg (twice, separate processes) and c3_sweep.py (twice)
for i in 1 2; do
  python bench.py --steps 5 --no-cpu-baseline --no-training --no-e2e > gpurun_out/bv$i.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/bv$i.json'))['roofline_fine_sweep_c3']; print('bench leg', round(d['ms_per_sweep'],3), round(d['frac'],3))"
  python scripts/c3_sweep.py
done
