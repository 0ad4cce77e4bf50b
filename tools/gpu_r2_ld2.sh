# A/B on one box: in-tree library vs variants/ld2.so (Vn / T loaded per step instead of one step ahead)
mkdir -p gpurun_out
for cfg in c4 c3 c5slab-med c5slab-low c2; do
  echo "LIB $(timeout 300 python tools/kbench.py $cfg 0.05)"
  echo "LD2 $(ODP_LIB_PATH=variants/ld2.so timeout 300 python tools/kbench.py $cfg 0.05)"
done 2>&1 | tee gpurun_out/ld2_kbench.log
