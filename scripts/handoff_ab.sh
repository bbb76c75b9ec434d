# pipelined schedule, fine(k, k−1) reading F̂ directly (new) vs via the chain's copy (old):
# the pipe tests on the new build, then interleaved bench medians of both builds on one box
O=gpurun_out/handoff; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "pipelined or headline or graph or determinism or pinn_fixed or co_resident or device_entry" 2>&1 | tail -5 > $O/pytest.txt; cat $O/pytest.txt
for rep in 1 2 3; do
  for v in old new; do
    for a in "" "--pinn-width 50 --pinn-layers 10" "--coarse ie"; do
      PR_LIB_VARIANT=paper_2303_03848_b200/libparareal_$v.so timeout 300 python bench.py $a --no-cpu-baseline --no-training --no-c3-sweep --no-e2e 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print('$rep $v [$a]', round(d['step_ms_stats']['median'],4), round(d['ms_per_step'],4))"
    done
  done
done 2>&1 | tee $O/ab.txt
timeout 120 python scripts/pipe_trace.py > $O/pipe_trace.txt 2>&1; head -20 $O/pipe_trace.txt
