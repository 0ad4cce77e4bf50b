set -x
for v in variants/*.so; do
  echo "== $v"
  ODP_LIB_PATH=$v python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
  for c in ${CFGS:-c4 c3 c2}; do ODP_LIB_PATH=$v timeout 300 python tools/kbench.py $c 0.05 2>&1 | tail -1; done
done
