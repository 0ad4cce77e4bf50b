for b in 1 2 3 5 6 10 15 30; do echo "== B1=$b"; ODP_MARCH_B1=$b timeout 300 python tools/kbench.py c4 0.2 2>&1 | tail -1; done
for b in 1 3 6 12 24 48; do echo "== c5low B1=$b"; ODP_MARCH_B1=$b timeout 300 python tools/kbench.py c5slab-low 0.2 2>&1 | tail -1; done
