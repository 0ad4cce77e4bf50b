for lib in tools/libodp_lean0.so ""; do
  echo "== lib ${lib:-lean (default)}"
  for cfg in c4 c3 c2 c5slab-low c5slab-med; do ODP_LIB_PATH=$lib timeout 300 python tools/kbench.py $cfg 0.2 2>&1 | tail -1; done
done
timeout 900 python -m pytest -q -x tests/test_gpu_march.py tests/test_gpu_checked.py tests/test_gpu_loopback.py tests/test_gpu_edges.py 2>&1 | tail -2
timeout 900 python -m pytest -q -x tests/test_gpu_parity.py -k "march" 2>&1 | tail -2
