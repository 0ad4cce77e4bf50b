# full GPU test suite + default-plan timing of every HJ config
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
for cfg in c4 c5slab-low c5slab-med c3 c2 c1 f2; do timeout 300 python tools/kbench.py $cfg 0.05; done
timeout 3000 python -m pytest -q tests -m gpu -x --durations=15 2>&1 | tail -40
