set -x
for L2 in 0 24e6 48e6 96e6; do
  ODP_TILED_L2_BYTES=$L2 python tools/kbench.py c4 0.05 2>&1 | tail -1
  ODP_TILED_L2_BYTES=$L2 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sector_hit_rate.pct,lts__t_bytes.sum -k regex:k_tiled -c 2 python tools/profile_run.py c4 0.02 2>&1 | grep -E "k_tiled|duration|dram__|lts__" | head -12
done
