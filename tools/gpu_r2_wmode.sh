for lib in w1p1 w1p2 w2p2 w3p3; do
  for d in 0 6; do
    echo "== $lib DBG=$d"
    ODP_LIB_PATH=tools/libodp_$lib.so ODP_MARCH_DBG=$d ODP_MARCH_B=30 ODP_MARCH_NST=2 timeout 300 python tools/kbench.py c4 0.2 2>&1 | grep stages | tail -1
    ODP_LIB_PATH=tools/libodp_$lib.so ODP_MARCH_DBG=$d timeout 300 python tools/kbench.py c5slab-low 0.2 2>&1 | grep stages | tail -1
  done
done
