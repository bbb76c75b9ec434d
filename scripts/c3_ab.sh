# A/B of two library builds (PR_LIB_VARIANT) on one box: bench C3 leg and c3_sweep.py, alternating
for v in packed s32 packed s32; do
  PR_LIB_VARIANT=paper_2303_03848_b200/libparareal_$v.so python scripts/c3_sweep.py | sed "s/^/$v /"
  PR_LIB_VARIANT=paper_2303_03848_b200/libparareal_$v.so python bench.py --steps 5 --no-cpu-baseline --no-training --no-e2e > gpurun_out/bab.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/bab.json'))['roofline_fine_sweep_c3']; print('$v bench leg', round(d['ms_per_sweep'],3), round(d['frac'],3))"
done
