# round 2: march pipeline depth sweep (issue-ahead producer, rdy barriers)
mkdir -p gpurun_out
timeout 900 python -m pytest -q -x tests/test_gpu_march.py tests/test_gpu_parity.py -k "march or auto" 2>&1 | tail -3
run() { echo "== $*"; env "$@" timeout 300 python tools/kbench.py $CFG 0.05; }
CFG=c4; run ODP_MARCH_NST=2; run ODP_MARCH_NST=3 ODP_MARCH_B=10; run ODP_MARCH_NST=4 ODP_MARCH_B=10
CFG=c5slab-low; run ODP_MARCH_NST=2; run ODP_MARCH_NST=3; run ODP_MARCH_NST=4; run ODP_MARCH_NST=4 ODP_MARCH_B=8
CFG=c5slab-med; run ODP_MARCH_NST=2; run ODP_MARCH_NST=3; run ODP_MARCH_NST=4 ODP_MARCH_B=8
CFG=c3; run ODP_MARCH_NST=2; run ODP_MARCH_NST=3; run ODP_MARCH_NST=4 ODP_MARCH_B=10
CFG=c2; run ODP_MARCH_NST=2; run ODP_MARCH_NST=3; run ODP_MARCH_NST=4
CFG=c1; run ODP_MARCH_NST=2; run ODP_MARCH_NST=3
