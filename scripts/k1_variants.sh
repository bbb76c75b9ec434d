# K1 variants: GPU tests, then the C2 CN, paper-net and C4 bench lines (short)
O=gpurun_out/k1v; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
for a in "--fine-theta 0.5" "--pinn-width 50 --pinn-layers 10" "--config C4 --steps 5" "--coarse ie"; do
  timeout 300 python bench.py $a --no-cpu-baseline --no-training --no-c3-sweep --no-e2e > $O/b.json 2>/dev/null
  python -c "import json; d=json.load(open('$O/b.json')); print('$a', round(d['ms_per_step'],4), round(d['step_ms_stats']['median'],4), 'serial', round(d.get('serial_fine_ms') or 0,3), 'speedup', round(d.get('speedup_vs_serial_fine') or 0,2))"
done
