# One bench line per HJ config (no CPU baseline): value, roofline fractions, single-pass variant
for c in c1 c2 c3 c4 f2 c5slab-low c5slab-med; do
  timeout 600 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); r=d['roofline']; sp=d.get('single_pass') or {}
print(f\"{d['config']['workload']:12s} grid {'x'.join(map(str,d['config']['grid'])):22s} {d['config']['accuracy']:6s} {d['value']/1e9:8.2f} Gpt-st/s  dominant frac {r['frac']:.3f}  stage frac {(r.get('stage') or {}).get('frac', r['frac']):.3f}  issue {((r.get('issue') or {}).get('frac') or 0):.2f}  single-pass {sp.get('value',0)/1e9:8.2f} (bitwise {sp.get('bitwise_equal_to_two_pass')})  kernel {d['config']['kernel']}\")
" || echo "$c failed"
done
