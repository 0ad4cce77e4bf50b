# HEAD check, part 2: the secondary bench lines (f2, c1, t1, v2) and the ncu launch list of tools/profile_run.py c4 0.05 (as r02f)
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv,noheader
for cfg in f2 c1 t1 v2; do
  timeout 400 python bench.py --config $cfg > gpurun_out/head_bench_$cfg.json 2> gpurun_out/head_bench_$cfg.err; echo "bench_${cfg}_rc=$?"
  cat gpurun_out/head_bench_$cfg.json
done
timeout 300 python tools/profile_run.py c4 0.05 > gpurun_out/head_b2.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/head_launches.csv python tools/profile_run.py c4 0.05 > gpurun_out/head_ncu.log 2>&1
echo "ncu_rc=$?"; wc -l gpurun_out/head_launches.csv
