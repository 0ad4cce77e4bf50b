# round 2 iteration: march-kernel parity + per-pass timing of the HJ configs
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
timeout 1200 python -m pytest -q -x tests/test_gpu_march.py tests/test_gpu_parity.py -k "march or auto" 2>&1 | tail -15
for cfg in c4 c5slab-low c5slab-med c3 c2 c1; do timeout 300 python tools/kbench.py $cfg 0.05; done
for B in 15; do echo "B=$B"; ODP_MARCH_B=$B timeout 300 python tools/kbench.py c4 0.05; done
