# Round profile: bench line, ncu launch list, ncu --set full of the two hot kernels.  Writes gpurun_out/.
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv,noheader
python bench.py --steps ${STEPS:-3} --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -2 gpurun_out/bench.err
cat gpurun_out/bench.json
python tools/profile_run.py c4 0.05 > gpurun_out/plain_prof.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python tools/profile_run.py c4 0.05 > gpurun_out/ncu_launches.log 2>&1
tail -1 gpurun_out/ncu_launches.log
ncu --set full --clock-control none --import-source on -k regex:${KREGEX:-k_march} -s 0 -c 2 -o gpurun_out/prof_full python tools/profile_run.py c4 0.02 > gpurun_out/ncu_full.log 2>&1
tail -1 gpurun_out/ncu_full.log
