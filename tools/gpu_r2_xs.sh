# A/B: pass 2's T / Vn staged by TMA (variants/xs.so default) vs per-thread global loads (ODP_MARCH_XS=0)
mkdir -p gpurun_out
export ODP_LIB_PATH=variants/xs.so
for cfg in c4 c5slab-low c5slab-med c3 c2; do
  timeout 300 python tools/kbench.py $cfg 0.05
  ODP_MARCH_XS=0 timeout 300 python tools/kbench.py $cfg 0.05
done 2>&1 | tee gpurun_out/xs_kbench.log
timeout 1200 python -m pytest -q -x tests/test_gpu_parity.py tests/test_gpu_edges.py tests/test_gpu_march.py tests/test_gpu_loopback.py tests/test_gpu_dist.py \
  "tests/test_gpu_parity_full.py::test_c5_slab_low_one_step" "tests/test_gpu_parity_full.py::test_c2_full_size_full_horizon" \
  "tests/test_gpu_parity_full.py::test_medium_full_size_full_horizon_sampled" 2>&1 | tail -5
