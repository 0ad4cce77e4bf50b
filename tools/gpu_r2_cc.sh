# ncu launch list of the c4 march kernels with and without ncu's cache flush (why ncu's per-launch
# times are ~20 % below the live CUDA-event times)
mkdir -p gpurun_out
python tools/profile_run.py c4 0.02 > /dev/null 2>&1
for cc in all none; do
  ncu --metrics gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second,dram__cycles_elapsed.avg.per_second --clock-control none --cache-control $cc -k regex:k_march -c 6 --csv --log-file gpurun_out/cc_$cc.csv python tools/profile_run.py c4 0.02 > /dev/null 2>&1
  echo "== cache-control $cc"; grep -E 'time_duration|per_second' gpurun_out/cc_$cc.csv | awk -F'","' '{print $5, $(NF-2), $(NF-1), $NF}' | cut -c1-200
done
