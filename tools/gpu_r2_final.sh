# Round-2 final: GPU suite, smoke, the default bench line, one bench line per HJ config, launch list of c4
mkdir -p gpurun_out
T=${TAG:-r02c}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv,noheader
timeout 2400 python -m pytest -q tests -m gpu -x --durations=15 -rs > gpurun_out/${T}_pytest.log 2>&1; echo "pytest_rc=$?"
tail -25 gpurun_out/${T}_pytest.log
timeout 600 python -m pytest -q -s "tests/test_gpu_parity_full.py::test_medium_full_size_full_horizon_sampled" 2>&1 | grep -E 'nodes|passed|failed' | tee gpurun_out/${T}_sampled.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.log 2>&1; echo "smoke_rc=$?"
python bench.py --steps 10 --warmup 3 > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err; echo "bench_rc=$?"
cat gpurun_out/${T}_bench.json
bash tools/bench_configs.sh > gpurun_out/${T}_configs.txt 2>&1; cat gpurun_out/${T}_configs.txt
python tools/profile_run.py c4 0.05 > gpurun_out/plain_launch.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${T}_launches.csv python tools/profile_run.py c4 0.05 > gpurun_out/ncu_launches.log 2>&1
tail -1 gpurun_out/ncu_launches.log

