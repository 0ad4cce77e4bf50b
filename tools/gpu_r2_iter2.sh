mkdir -p gpurun_out
timeout 900 python -m pytest -q -x tests/test_gpu_march.py tests/test_gpu_parity.py tests/test_gpu_loopback.py -k "march or auto or loopback" 2>&1 | tail -3
for cfg in c4 c5slab-low c5slab-med c3 c2 c1; do timeout 300 python tools/kbench.py $cfg 0.05; done
