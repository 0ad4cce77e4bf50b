# k_amax3_fin (range + alpha^max + finalize in one launch, DEPS3 on one rank): tests and f2 bench
mkdir -p gpurun_out
[ -n "$TESTS" ] && timeout 900 python -m pytest -q tests/test_gpu_pairdubins.py tests/test_gpu_resident.py -x 2>&1 | tail -3
for env in "ODP_AMAX3_SPLIT=1 ODP_AMAX3_CPS=2" "ODP_AMAX3_CPS=2" "ODP_AMAX3_SPLIT=1 ODP_AMAX3_CPS=4" "ODP_AMAX3_CPS=4" "ODP_AMAX3_SPLIT=1 ODP_AMAX3_CPS=6" "ODP_AMAX3_CPS=6" "ODP_AMAX3_CPS=3"; do
  echo "== f2 $env"
  env $env timeout 300 python bench.py --config f2 --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value']/1e9, 'Gpt-st/s', d['ms_per_step'], 'ms/solve', d['gpu_launches'], 'launches', d['kernel_ms_share'])"
done
