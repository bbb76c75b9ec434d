# A/B of library builds (PR_LIB_VARIANT) on one box: headline and paper-net bench medians
for v in $VARIANTS; do
  for a in "" "--pinn-width 50 --pinn-layers 10"; do
    PR_LIB_VARIANT=paper_2303_03848_b200/libparareal_$v.so python bench.py $a --no-cpu-baseline --no-training --no-c3-sweep --no-e2e 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print('$v', '$a', d['step_ms_stats']['median'])"
  done
done
