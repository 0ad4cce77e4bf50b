# round 2: march geometry sweep (segment length K, axis-1 work-order block B1) on c4 + sanity tests
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv,noheader
timeout 900 python -m pytest -q -x tests/test_gpu_vi.py tests/test_gpu_ttr.py 2>&1 | tail -3
for cfg in c4 c5slab-low c2; do python tools/kbench.py $cfg 0.05; done
for K in 15 10 6 4; do echo "K=$K"; ODP_MARCH_K=$K python tools/kbench.py c4 0.05; done
for B1 in 1 3 10 30; do echo "B1=$B1"; ODP_MARCH_B1=$B1 python tools/kbench.py c4 0.05; done
for K in 10 6; do for B1 in 3 10; do echo "K=$K B1=$B1"; ODP_MARCH_K=$K ODP_MARCH_B1=$B1 python tools/kbench.py c4 0.05; done; done
