# quick timing sweep of march-family env knobs on c4: bash tools/gpu_sweep.sh "ODP_MARCH_K=30" "ODP_MARCH_K=10" ...
for cfg in "$@"; do
  env $cfg timeout 300 python bench.py --steps 2 --warmup 1 --no-cpu-baseline --kernel march 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$cfg', round(d['value']/1e9,2), 'Gpt-st/s', round(d['ms_per_step'],1), 'ms/solve; pass2', round(d['roofline']['avg_launch_ms'],3), 'pass1', round(d['roofline']['stage']['pass1_ms'],3))"
done
if [ -n "$NCUDRAM" ]; then
  env $NCUDRAM ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k_march -c 4 python tools/profile_run.py c4 0.02 march 2>&1 | grep -E "k_march|dram__|gpu__time" | head -20
fi
