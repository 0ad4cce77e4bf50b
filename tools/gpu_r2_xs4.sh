# A/B on one box: HEAD library vs variants/xs4.so (and xs4 with ODP_MARCH_XS=0: pass-1 tile skip only)
mkdir -p gpurun_out
for cfg in c5slab-low c4 c3 c2 c5slab-med; do
  echo "HEAD $(timeout 300 python tools/kbench.py $cfg 0.05)"
  echo "XS4  $(ODP_LIB_PATH=variants/xs4.so timeout 300 python tools/kbench.py $cfg 0.05)"
  echo "XS4/0 $(ODP_MARCH_XS=0 ODP_LIB_PATH=variants/xs4.so timeout 300 python tools/kbench.py $cfg 0.05)"
done 2>&1 | tee gpurun_out/xs4_kbench.log
export ODP_LIB_PATH=variants/xs4.so
timeout 1200 python -m pytest -q -x tests/test_gpu_parity.py tests/test_gpu_edges.py tests/test_gpu_march.py tests/test_gpu_loopback.py tests/test_gpu_dist.py \
  "tests/test_gpu_parity_full.py::test_c5_slab_low_one_step" "tests/test_gpu_parity_full.py::test_c2_full_size_full_horizon" 2>&1 | tail -3
