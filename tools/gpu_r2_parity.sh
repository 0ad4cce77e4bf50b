# round 2: new parity / loopback / single-pass tests
mkdir -p gpurun_out
timeout 2400 python -m pytest -q tests/test_gpu_dist.py tests/test_gpu_edges.py tests/test_gpu_pairdubins.py tests/test_gpu_parity_full.py -s -k "not c2_full and not c5_slab_low and not one_and_two" 2>&1 | grep -v "^$" | tail -30
timeout 2400 python -m pytest -q tests/test_gpu_parity.py -k "medium" 2>&1 | tail -5
