mkdir -p gpurun_out
timeout 900 python -m pytest -q -x tests/test_gpu_march.py tests/test_gpu_parity.py tests/test_gpu_loopback.py tests/test_gpu_dist.py -k "march or auto or loopback or single_pass" 2>&1 | tail -3
for rp in 1 2; do echo "== RP=$rp"; for cfg in c4 c5slab-low c5slab-med c3 c2; do ODP_MARCH_RP=$rp timeout 300 python tools/kbench.py $cfg 0.05; done; done
