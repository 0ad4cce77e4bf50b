# small grids: march geometry for more units (c1 41x41x36, f2 100^3)
for cfg in c1 f2; do
  for b in "" 2 4 6 10; do for k in "" 2 4 8; do
    echo "== $cfg B=${b:-auto} K=${k:-auto}"; ODP_MARCH_B=$b ODP_MARCH_K=$k ODP_MARCH_NST=2 timeout 120 python tools/kbench.py $cfg 0.2 2>&1 | tail -1
  done; done
done
python bench.py --config c1 --steps 5 --warmup 3 --no-cpu-baseline --single-pass-too 0 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('bench c1', d['value'], d['ms_per_step'])"
