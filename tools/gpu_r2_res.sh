timeout 900 python -m pytest -q -x tests/test_gpu_resident.py 2>&1 | tail -3
timeout 900 python -m pytest -q -x tests/test_gpu_parity.py -k "resident or generic" 2>&1 | tail -3
for c in c1 c2; do timeout 300 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c', d['value'], d['ms_per_step'], d.get('e2e',{}).get('value'), d.get('gpu_launches'))"; done
