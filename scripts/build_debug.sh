# Test-only library variant with device-side index checks (-DPR_DEBUG_BOUNDS: trap on violation),
# compute-sanitizer being closed on the GPU pool: PR_LIB_VARIANT=paper_2303_03848_b200/libparareal_dbg.so
set -e
mkdir -p build_dbg
for u in parareal res streamed pinn_smem pinn_param misc pipe pinn_tc pinn_train fine_grid; do
  nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo -Xcompiler -fPIC -DPR_DEBUG_BOUNDS \
       -c -o build_dbg/$u.o paper_2303_03848_b200/csrc/$u.cu &
done
wait
nvcc -shared -gencode arch=compute_100a,code=sm_100a -cudart static -ldl -o paper_2303_03848_b200/libparareal_dbg.so build_dbg/*.o
