# usage: bash tools/gpu_check.sh [pytest-args...]
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -3
timeout 1200 python -m pytest tests -m gpu -q "$@" 2>&1 | tail -25
timeout 600 python bench.py --steps 3 --warmup 1 --no-cpu-baseline > gpurun_out/bench_auto.json 2> gpurun_out/bench_auto.err; tail -3 gpurun_out/bench_auto.err; cat gpurun_out/bench_auto.json
