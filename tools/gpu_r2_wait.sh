# wait-strategy variants of the march kernels (compute warps waiting on the TMA barrier)
for lib in "" tools/libodp_wait0_64.so tools/libodp_wait0_256.so; do
  echo "== lib ${lib:-default}"
  for cfg in c4 c5slab-low c3 c2; do ODP_LIB_PATH=$lib timeout 300 python tools/kbench.py $cfg 0.05; done
done
