# c4 bench under several march geometries (ODP_MARCH_B / ODP_MARCH_NST); one line each
for cfg in "30 2" "15 2" "10 2" "15 3" "10 3" "10 4" "30 3"; do
  set -- $cfg
  ODP_MARCH_B=$1 ODP_MARCH_NST=$2 timeout 300 python bench.py --steps 2 --warmup 1 --no-cpu-baseline --single-pass-too 0 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('B=$1 NST=$2', round(d['value']/1e9,2), 'Gpt-st/s; pass2', round(d['roofline']['avg_launch_ms'],3), 'pass1', round(d['roofline']['stage']['pass1_ms'],3))" || echo "B=$1 NST=$2 failed"
done
