# round-2 GPU run 1: peaks microbenchmark, GPU tests, smoke, default bench, ncu source capture of
# the K2 pass at C3, compute-sanitizer on the small cases of every kernel family
set -x
mkdir -p gpurun_out/r02
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
./scripts/peaks > gpurun_out/r02/peaks.json 2>&1; cat gpurun_out/r02/peaks.json
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -25 > gpurun_out/r02/pytest.txt; tail -5 gpurun_out/r02/pytest.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02/smoke.txt 2>&1; tail -3 gpurun_out/r02/smoke.txt
timeout 900 python bench.py > gpurun_out/r02/bench_default.json 2> gpurun_out/r02/bench_default.err; tail -c 600 gpurun_out/r02/bench_default.err
for c in c1pipe c2num k2res k4 c4; do
  for t in memcheck racecheck synccheck; do
    timeout 300 compute-sanitizer --tool $t --print-limit 20 python scripts/sanitize_target.py $c > gpurun_out/r02/san_${c}_${t}.txt 2>&1
    echo "$c $t rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' gpurun_out/r02/san_${c}_${t}.txt | tail -1)"
  done
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_pass_res2 -s 4 -c 2 -o gpurun_out/r02/prof_k2res2 python scripts/prof_target.py c3 > gpurun_out/r02/prof_k2res2.log 2>&1; tail -3 gpurun_out/r02/prof_k2res2.log
ls -la gpurun_out/r02
