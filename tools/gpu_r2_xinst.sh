# c5-slab LOW row-block size: B = 16 (2 CTAs/SM, default) vs 12 / 8 (3-4 CTAs/SM), variants/xinst.so
mkdir -p gpurun_out
export ODP_LIB_PATH=variants/xinst.so
for B in 16 12 8; do
  for XS in 1 0; do
    echo "B=$B XS=$XS $(ODP_MARCH_VERBOSE=1 ODP_MARCH_XS=$XS ODP_MARCH_B=$B timeout 300 python tools/kbench.py c5slab-low 0.05 2>&1 | grep -E 'plan|stages' | sort -u | tr '\n' ' ')"
  done
done 2>&1 | tee gpurun_out/xinst_kbench.log
