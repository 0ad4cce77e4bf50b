# Round-2 profile: bench line (c4), ncu launch list of c4, ncu --set full of one time step of c4
# (MEDIUM: 4 march launches) and c5-slab LOW (2 launches).  Writes gpurun_out/; summaries are made
# on the CPU side with tools/ncu_kernels.py and tools/make_profiles.py.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv,noheader
python bench.py --steps ${STEPS:-10} --warmup 3 > gpurun_out/${TAG:-r02}_bench.json 2> gpurun_out/${TAG:-r02}_bench.err; tail -2 gpurun_out/${TAG:-r02}_bench.err
cat gpurun_out/${TAG:-r02}_bench.json
python tools/profile_run.py c4 0.05 > gpurun_out/plain_launch.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${TAG:-r02}_launches.csv python tools/profile_run.py c4 0.05 > gpurun_out/ncu_launches.log 2>&1
tail -1 gpurun_out/ncu_launches.log
python tools/profile_run.py c4 0.01 > gpurun_out/plain_c4.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_march -c 4 -o gpurun_out/${TAG:-r02}_c4 python tools/profile_run.py c4 0.01 > gpurun_out/ncu_c4.log 2>&1
tail -1 gpurun_out/ncu_c4.log
python tools/profile_run.py c5slab-low 0.01 > gpurun_out/plain_low.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_march -c 2 -o gpurun_out/${TAG:-r02}_c5low python tools/profile_run.py c5slab-low 0.01 > gpurun_out/ncu_low.log 2>&1
tail -1 gpurun_out/ncu_low.log
# keep the call's output under gpurun's 64 MiB: raw metric pages and SASS source pages as CSV
for r in ${TAG:-r02}_c4 ${TAG:-r02}_c5low; do
  ncu -i gpurun_out/$r.ncu-rep --page raw --csv --print-units base > gpurun_out/${r}_raw.csv 2>/dev/null
  ncu -i gpurun_out/$r.ncu-rep --page raw --csv > gpurun_out/${r}_raw_units.csv 2>/dev/null
  ncu -i gpurun_out/$r.ncu-rep --page source --csv --print-source sass > gpurun_out/${r}_sass.csv 2>/dev/null
done
gzip -f gpurun_out/*_sass.csv
rm -f gpurun_out/${TAG:-r02}_c5low.ncu-rep gpurun_out/${TAG:-r02}_c4.ncu-rep
ls -la gpurun_out/
