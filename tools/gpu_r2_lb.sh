export ODP_LIB_PATH=tools/libodp_exp.so ODP_MARCH_VERBOSE=1
run() { echo "== $*"; env "$@" timeout 300 python tools/kbench.py c4 0.2 2>&1 | grep -v "^$" | sort | uniq | tail -4; }
run X=0
run ODP_MARCH_1CTA=1 ODP_MARCH_NST=4
run ODP_MARCH_B=15 ODP_MARCH_NST=2
run ODP_MARCH_B=10 ODP_MARCH_NST=3
run ODP_MARCH_B=10 ODP_MARCH_NST=2
