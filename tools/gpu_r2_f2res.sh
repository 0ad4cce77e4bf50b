# f2 (Eq. 7, 100^3) through the resident kernel: tests, then bench with the launch path vs resident
mkdir -p gpurun_out
timeout 900 python -m pytest -q tests/test_gpu_resident.py tests/test_gpu_pairdubins.py -x 2>&1 | tail -5
for env in "ODP_RESIDENT_MAX_POINTS=1" "ODP_RESIDENT_MAX_POINTS=2000000"; do
  echo "== f2 $env"
  env $env timeout 300 python bench.py --config f2 --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value']/1e9, 'Gpt-st/s', d['ms_per_step'], 'ms/solve', d['gpu_launches'], 'launches', d['roofline']['kernel'])"
done
echo "== c1"; timeout 300 python bench.py --config c1 --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value']/1e9, 'Gpt-st/s', d['ms_per_step'], 'ms/solve', d['gpu_launches'])"
