# experiment timings: bash tools/gpu_exp.sh "ENV1" "ENV2" ... (each: env assignments for exp_time.py)
for cfg in "$@"; do
  echo "== $cfg"; env $cfg timeout 120 python tools/exp_time.py c4 2>&1 | tail -1
done
