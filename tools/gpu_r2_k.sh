for k in 30 15 10 6; do for b in 3 30; do echo "== K=$k B1=$b"; ODP_MARCH_K=$k ODP_MARCH_B1=$b timeout 300 python tools/kbench.py c4 0.2 2>&1 | tail -1; done; done
for k in 48 24 16; do echo "== c5low K=$k"; ODP_MARCH_K=$k timeout 300 python tools/kbench.py c5slab-low 0.2 2>&1 | tail -1; done
