export ODP_MARCH_VERBOSE=1
for c in c4 c3 c2 c5slab-low c5slab-med; do timeout 300 python tools/kbench.py $c 0.2 2>&1 | grep -v "^$" | sort -u | tail -2; done
timeout 1200 python -m pytest -q -x tests/test_gpu_march.py tests/test_gpu_parity.py -k "march or auto" 2>&1 | tail -3
