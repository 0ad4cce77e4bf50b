# ncu --set full of the two march kernels of a config under the current env knobs
mkdir -p gpurun_out
python tools/profile_run.py ${CFG:-c4} 0.02 > gpurun_out/plain_${TAG}.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_march -s 2 -c 2 -o gpurun_out/prof_${TAG} python tools/profile_run.py ${CFG:-c4} 0.02 > gpurun_out/ncu_${TAG}.log 2>&1
tail -1 gpurun_out/ncu_${TAG}.log
