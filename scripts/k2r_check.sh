# K2R variant check: grid parity tests, C3-grid sweep tests, grid trace, C3 sweep time, grid_vs_k2 at 2^20
O=gpurun_out/k2r; mkdir -p $O
timeout 600 python -m pytest tests -m gpu -q -k "grid or c3 or C3" 2>&1 | tail -5 > $O/pytest.txt; cat $O/pytest.txt
timeout 120 python scripts/grid_trace.py > $O/grid_trace.txt 2>&1; cat $O/grid_trace.txt
FINE_KERNEL=3 timeout 300 python scripts/c3_sweep.py > $O/c3_sweep.txt 2>&1; cat $O/c3_sweep.txt
[ -n "$VS" ] && timeout 300 python scripts/grid_vs_k2.py > $O/grid_vs_k2.txt 2>&1; cat $O/grid_vs_k2.txt
