# A/B on one box: variants/xs4.so vs xs5.so (compile-time dbg, Euler for R = 1, CT marching table); c2 segment-length sweep
mkdir -p gpurun_out
for cfg in c5slab-low c4 c3 c2 c5slab-med; do
  echo "XS4 $(ODP_LIB_PATH=variants/xs4.so timeout 300 python tools/kbench.py $cfg 0.05)"
  echo "XS5 $(ODP_LIB_PATH=variants/xs5.so timeout 300 python tools/kbench.py $cfg 0.05)"
done 2>&1 | tee gpurun_out/xs5_kbench.log
for K in 6 8 10 12 15 20 30 60; do echo "K=$K $(ODP_MARCH_K=$K ODP_LIB_PATH=variants/xs5.so timeout 300 python tools/kbench.py c2 0.1)"; done 2>&1 | tee -a gpurun_out/xs5_kbench.log
for K in 10 20 40; do echo "c3 K=$K $(ODP_MARCH_K=$K ODP_LIB_PATH=variants/xs5.so timeout 300 python tools/kbench.py c3 0.05)"; done 2>&1 | tee -a gpurun_out/xs5_kbench.log
export ODP_LIB_PATH=variants/xs5.so
timeout 1200 python -m pytest -q -x tests/test_gpu_parity.py tests/test_gpu_edges.py tests/test_gpu_march.py tests/test_gpu_loopback.py tests/test_gpu_dist.py \
  "tests/test_gpu_parity_full.py::test_c5_slab_low_one_step" "tests/test_gpu_parity_full.py::test_c2_full_size_full_horizon" 2>&1 | tail -3
