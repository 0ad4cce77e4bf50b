for lib in "" tools/libodp_pd150.so tools/libodp_pd400.so; do
  echo "== lib ${lib:-default}"
  for cfg in c4 c5slab-low; do ODP_LIB_PATH=$lib timeout 300 python tools/kbench.py $cfg 0.2 2>&1 | tail -1; done
done
