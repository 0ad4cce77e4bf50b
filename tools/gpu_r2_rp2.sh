export ODP_LIB_PATH=tools/libodp_rp.so ODP_MARCH_VERBOSE=1
timeout 600 python tools/rp_check.py 2>&1 | grep -v "march plan" | tail -3
for rp in 1 2; do echo "== RP=$rp"; ODP_MARCH_RP=$rp timeout 300 python tools/kbench.py c4 0.2 2>&1 | sort -u | tail -2; done
