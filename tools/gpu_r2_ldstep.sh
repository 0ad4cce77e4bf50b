# A/B on one box: in-tree library vs variants/ldstep.so (MEDIUM pass 2 compiled + RK2 per-step Vn/T loads)
mkdir -p gpurun_out
for rep in 1 2; do
for cfg in c4 c3 c5slab-med; do
  echo "LIB   $(timeout 300 python tools/kbench.py $cfg 0.05)"
  echo "LDSTEP $(ODP_LIB_PATH=variants/ldstep.so timeout 300 python tools/kbench.py $cfg 0.05)"
done
done 2>&1 | tee gpurun_out/ldstep_kbench.log
export ODP_LIB_PATH=variants/ldstep.so
timeout 1200 python -m pytest -q -x tests/test_gpu_parity.py tests/test_gpu_edges.py "tests/test_gpu_parity_full.py::test_medium_full_size_one_and_two_steps" \
   "tests/test_gpu_parity_full.py::test_medium_full_size_full_horizon_sampled" tests/test_gpu_loopback.py 2>&1 | tail -3
