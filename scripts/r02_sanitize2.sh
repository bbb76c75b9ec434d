# compute-sanitizer after the K1 zig-zag and trainer v2 changes
mkdir -p gpurun_out/r02s
for c in c1pipe c2num c4 train; do
  for t in memcheck racecheck synccheck; do
    timeout 300 compute-sanitizer --tool $t --print-limit 20 python scripts/sanitize_target.py $c > gpurun_out/r02s/san_${c}_${t}.txt 2>&1
    echo "$c $t rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' gpurun_out/r02s/san_${c}_${t}.txt | tail -1)"
  done
done
