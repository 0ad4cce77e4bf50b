# A/B on one box: HEAD library vs variants/xs3.so (LOW pass 2 T staged by TMA, LOW pass 1 without the -1 side tile)
mkdir -p gpurun_out
for rep in 1 2; do
for cfg in c5slab-low c2 c4 c3 c5slab-med; do
  echo "HEAD $(timeout 300 python tools/kbench.py $cfg 0.05)"
  echo "XS3  $(ODP_LIB_PATH=variants/xs3.so timeout 300 python tools/kbench.py $cfg 0.05)"
done
done 2>&1 | tee gpurun_out/xs3_kbench.log
ODP_MARCH_VERBOSE=1 ODP_LIB_PATH=variants/xs3.so python tools/kbench.py c5slab-low 0.01 2>&1 | grep plan | head -2
ODP_MARCH_VERBOSE=1 ODP_LIB_PATH=variants/xs3.so python tools/kbench.py c4 0.01 2>&1 | grep plan | head -2
export ODP_LIB_PATH=variants/xs3.so
timeout 1200 python -m pytest -q -x tests/test_gpu_parity.py tests/test_gpu_edges.py tests/test_gpu_march.py tests/test_gpu_loopback.py tests/test_gpu_dist.py \
  "tests/test_gpu_parity_full.py::test_c5_slab_low_one_step" "tests/test_gpu_parity_full.py::test_c2_full_size_full_horizon" 2>&1 | tail -3
