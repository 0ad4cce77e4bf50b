mkdir -p gpurun_out
./tools/l2bw > gpurun_out/l2bw.txt 2>&1
python tools/profile_run.py c5slab-low 0.02 > gpurun_out/plain_low.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_march -s 2 -c 2 -o gpurun_out/prof_low python tools/profile_run.py c5slab-low 0.02 > gpurun_out/ncu_low.log 2>&1
tail -2 gpurun_out/ncu_low.log
