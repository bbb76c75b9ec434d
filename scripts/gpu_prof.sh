set -x
mkdir -p gpurun_out
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_streamed_pass -s 20 -c 2 -o gpurun_out/prof_streamed python scripts/prof_target.py c3 > gpurun_out/prof_streamed.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_pinn_chain -s 1 -c 1 -o gpurun_out/prof_pinn_c3 python scripts/prof_target.py c3 > gpurun_out/prof_pinn.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_fine_sweep -c 1 -o gpurun_out/prof_fine_c4 python scripts/prof_target.py c4 > gpurun_out/prof_fine.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_fine_sweep -c 1 -o gpurun_out/prof_fine_c2 python scripts/prof_target.py c2 > gpurun_out/prof_fine2.log 2>&1
ls -la gpurun_out
