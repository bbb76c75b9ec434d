# pipelined schedule: pipelined/headline/graph/determinism tests, the trace, a short bench
O=gpurun_out/pipe3; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "pipelined or headline or graph or determinism or pinn_fixed or k1_c2 or finite or device_entry or co_resident" 2>&1 | tail -5 > $O/pytest.txt; cat $O/pytest.txt
timeout 120 python scripts/pipe_trace.py > $O/pipe_trace.txt 2>&1; head -12 $O/pipe_trace.txt
timeout 600 python bench.py --no-cpu-baseline --no-training --no-c3-sweep > $O/bench.json 2> $O/bench.err; python -c "
import json; d=json.load(open('$O/bench.json')); print(d['ms_per_step'], d['step_ms_stats'], d['speedup_vs_serial_fine'], d['e2e'])"
