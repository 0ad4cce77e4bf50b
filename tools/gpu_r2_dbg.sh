for d in 0 4 2 6; do
  echo "== DBG=$d"
  for cfg in c4 c5slab-low; do ODP_LIB_PATH=tools/libodp_exp.so ODP_MARCH_DBG=$d timeout 300 python tools/kbench.py $cfg 0.2 2>&1 | grep stages | tail -1; done
done
