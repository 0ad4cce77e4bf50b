# usage: bash tools/gpu_march.sh  -- march-family parity + quick timing (run under gpurun)
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
python -c "import oracle; oracle.build()"
timeout 900 python -m pytest tests/test_gpu_march.py -x -q 2>&1 | tail -15
timeout 600 python -m pytest tests/test_gpu_parity.py -q -k "march or families" 2>&1 | tail -15
for k in march stream; do
  timeout 300 python bench.py --steps 2 --warmup 1 --no-cpu-baseline --kernel $k 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$k', d['value']/1e9, 'Gpt-st/s', d['ms_per_step'], 'ms', d['kernel_ms_share'], d['roofline']['avg_launch_ms'], d['roofline']['stage']['pass1_ms'])"
done
