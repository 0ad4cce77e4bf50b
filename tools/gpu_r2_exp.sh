# experiment: march kernels with the copies (DBG=4) or the arithmetic (DBG=2) switched off (garbage results)
for cfg in c4 c5slab-low; do for d in 0 2 4 6; do echo "DBG=$d"; ODP_LIB_PATH=tools/libodp_exp.so ODP_MARCH_DBG=$d timeout 300 python tools/exp_time.py $cfg; done; done
