# ncu --set full of the two march kernels on c4 (a few steps)
mkdir -p gpurun_out
python tools/profile_run.py c4 0.02 > gpurun_out/plain_c4.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_march -s 2 -c 2 -o gpurun_out/prof_${TAG:-new} python tools/profile_run.py c4 0.02 > gpurun_out/ncu_${TAG:-new}.log 2>&1
tail -2 gpurun_out/ncu_${TAG:-new}.log
