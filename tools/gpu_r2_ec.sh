for lib in "" tools/libodp_ec1.so tools/libodp_ec1n0.so tools/libodp_ec1n100.so; do
  echo "== lib ${lib:-default}"
  for cfg in c4 c3 c2 c5slab-low; do ODP_LIB_PATH=$lib timeout 300 python tools/kbench.py $cfg 0.2 2>&1 | tail -1; done
done
ODP_LIB_PATH=tools/libodp_ec1.so timeout 900 python -m pytest -q -x tests/test_gpu_march.py 2>&1 | tail -2
