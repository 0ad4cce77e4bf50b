# HEAD check: GPU suite (timed per test), smoke(), the default bench line, every HJ config's kernels
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv,noheader
timeout 2400 python -m pytest -q tests -m gpu -x --durations=25 > gpurun_out/head_pytest.log 2>&1; echo "pytest_rc=$?"
tail -40 gpurun_out/head_pytest.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/head_smoke.log 2>&1; echo "smoke_rc=$?"
python bench.py > gpurun_out/head_bench.json 2> gpurun_out/head_bench.err; echo "bench_rc=$?"; tail -3 gpurun_out/head_bench.err
cat gpurun_out/head_bench.json
for cfg in c4 c5slab-low c5slab-med c3 c2; do timeout 300 python tools/kbench.py $cfg 0.05; done > gpurun_out/head_kbench.log 2>&1
cat gpurun_out/head_kbench.log
