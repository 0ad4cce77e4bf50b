# ncu --set full of f2's kernels at HEAD: the fused range / alpha^max / finalize launch (k_amax3_fin) and the march passes
mkdir -p gpurun_out
python tools/profile_run.py f2 0.05 > gpurun_out/f2_plain.log 2>&1 && \
timeout 600 ncu --set full --clock-control none -k regex:"k_amax3|k_march" -s 6 -c 3 -f -o gpurun_out/prof_f2 python tools/profile_run.py f2 0.05 > gpurun_out/ncu_f2.log 2>&1
echo "ncu_rc=$?"; ls -la gpurun_out; tail -2 gpurun_out/f2_plain.log; tail -1 gpurun_out/ncu_f2.log
