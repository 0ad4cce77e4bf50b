# A/B: marching loop unrolled by 2 (variants/unroll2.so) vs the in-tree library; per-CUDA-line instruction counts of c4 pass 2
mkdir -p gpurun_out
for cfg in c4 c5slab-low c3 c2 c5slab-med; do
  echo "LIB $(timeout 300 python tools/kbench.py $cfg 0.05)"
  echo "UR2 $(ODP_LIB_PATH=variants/unroll2.so timeout 300 python tools/kbench.py $cfg 0.05)"
done 2>&1 | tee gpurun_out/unroll_kbench.log
python tools/profile_run.py c4 0.01 > /dev/null 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_march -s 1 -c 1 -o gpurun_out/c4p2 python tools/profile_run.py c4 0.01 > gpurun_out/ncu_c4p2.log 2>&1
python tools/ncu_cuda_lines.py gpurun_out/c4p2.ncu-rep k_march 80 > gpurun_out/c4p2_lines.txt 2>&1
ncu -i gpurun_out/c4p2.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/c4p2_cudasass.csv 2>/dev/null; gzip -f gpurun_out/c4p2_cudasass.csv
rm -f gpurun_out/c4p2.ncu-rep
head -50 gpurun_out/c4p2_lines.txt
