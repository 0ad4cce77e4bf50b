set -x
mkdir -p gpurun_out
K=${KREGEX:-k_stream}
python tools/profile_run.py c4 0.02 > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:$K -s 0 -c 2 -o gpurun_out/prof_c4 python tools/profile_run.py c4 0.02 > gpurun_out/ncu.log 2>&1
tail -2 gpurun_out/ncu.log
