# one compute-sanitizer tool per call (B200_PROFILING.md); TOOL=memcheck|racecheck|synccheck|initcheck
mkdir -p gpurun_out
python tools/sanitize_run.py > gpurun_out/san_plain.log 2>&1 && \
timeout 1500 compute-sanitizer --tool ${TOOL} --print-limit 20 python tools/sanitize_run.py > gpurun_out/san_${TOOL}.log 2>&1
tail -5 gpurun_out/san_${TOOL}.log
if [ -n "$BENCH" ]; then python bench.py --steps 10 --warmup 3 > gpurun_out/r02_bench.json 2> gpurun_out/r02_bench.err; tail -2 gpurun_out/r02_bench.err; fi
