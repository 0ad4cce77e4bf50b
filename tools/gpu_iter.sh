# one GPU iteration: march parity, quick bench (march vs stream), ncu of the two c4 march kernels
mkdir -p gpurun_out
python -c "import oracle; oracle.build()"
timeout 900 python -m pytest tests/test_gpu_march.py -x -q 2>&1 | tail -4
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_parity_full.py -x -q -k "march or families or full_size or one_and_two or slab" 2>&1 | tail -4
for k in march stream; do
  timeout 300 python bench.py --steps 2 --warmup 1 --no-cpu-baseline --kernel $k 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$k', round(d['value']/1e9,2), 'Gpt-st/s', round(d['ms_per_step'],1), 'ms/solve; pass2', round(d['roofline']['avg_launch_ms'],3), 'pass1', round(d['roofline']['stage']['pass1_ms'],3))"
done
if [ -n "$NCU" ]; then
python tools/profile_run.py c4 0.02 march > gpurun_out/plain.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:k_march -s 0 -c 2 -o gpurun_out/prof_$NCU python tools/profile_run.py c4 0.02 march > gpurun_out/ncu.log 2>&1; tail -1 gpurun_out/ncu.log
fi
