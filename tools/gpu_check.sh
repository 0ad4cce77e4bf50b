# usage: bash tools/gpu_check.sh [pytest-args...]
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -3
timeout 2400 python -m pytest tests -m gpu -q --durations=12 "$@" 2>&1 | tail -40
