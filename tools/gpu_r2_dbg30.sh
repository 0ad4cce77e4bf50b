for d in 0 4 2 6; do
  echo "== DBG=$d"
  ODP_LIB_PATH=tools/libodp_exp.so ODP_MARCH_DBG=$d ODP_MARCH_B=30 ODP_MARCH_NST=2 timeout 300 python tools/kbench.py c4 0.2 2>&1 | tail -1
  ODP_LIB_PATH=tools/libodp_exp.so ODP_MARCH_DBG=$d timeout 300 python tools/kbench.py c3 0.2 2>&1 | tail -1
done
