# interleaved bench medians of two library builds (old/new) on one box, default and paper net
O=gpurun_out/tail_ab; mkdir -p $O
for rep in 1 2 3 4; do
  for v in old new; do
    for a in "" "--pinn-width 50 --pinn-layers 10"; do
      PR_LIB_VARIANT=paper_2303_03848_b200/libparareal_$v.so timeout 300 python bench.py $a --no-cpu-baseline --no-training --no-c3-sweep --no-e2e 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print('$rep $v [$a]', round(d['step_ms_stats']['median'],4), round(d['ms_per_step'],4))"
    done
  done
done 2>&1 | tee $O/ab.txt
