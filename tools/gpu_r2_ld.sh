# A/B on one box: in-tree library vs variants/gh.so (cheaper column ghosts, LOW loop unrolled by 2) vs variants/ld.so
# (gh + Vn / T loaded per step instead of one step ahead)
mkdir -p gpurun_out
for cfg in c4 c5slab-low c3 c2 c5slab-med; do
  echo "LIB $(timeout 300 python tools/kbench.py $cfg 0.05)"
  echo "GH  $(ODP_LIB_PATH=variants/gh.so timeout 300 python tools/kbench.py $cfg 0.05)"
  echo "LD  $(ODP_LIB_PATH=variants/ld.so timeout 300 python tools/kbench.py $cfg 0.05)"
  echo "LD/XS0 $(ODP_MARCH_XS=0 ODP_LIB_PATH=variants/ld.so timeout 300 python tools/kbench.py $cfg 0.05)"
done 2>&1 | tee gpurun_out/ld_kbench.log
export ODP_LIB_PATH=variants/ld.so
timeout 1200 python -m pytest -q -x tests/test_gpu_parity.py tests/test_gpu_edges.py tests/test_gpu_march.py tests/test_gpu_loopback.py tests/test_gpu_dist.py \
  "tests/test_gpu_parity_full.py::test_c5_slab_low_one_step" "tests/test_gpu_parity_full.py::test_c2_full_size_full_horizon" \
  "tests/test_gpu_parity_full.py::test_medium_full_size_one_and_two_steps" 2>&1 | tail -3
