# rebuilt in-tree library: kernel timings and the march / checked / full-size LOW tests
mkdir -p gpurun_out
for cfg in c4 c5slab-low c3 c2 c5slab-med; do timeout 300 python tools/kbench.py $cfg 0.05; done 2>&1 | tee gpurun_out/verify_kbench.log
timeout 1500 python -m pytest -q -x tests/test_gpu_march.py tests/test_gpu_checked.py "tests/test_gpu_parity_full.py::test_c5_slab_low_one_step" 2>&1 | tail -3
