# Quick GPU pass: parity tests, smoke, then a short bench (no e2e / d100 / cpu baseline).
# usage: bash tools/gpu_quick.sh TAG [pytest -k expr]
TAG=${1:-quick}
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q ${2:+-k "$2"} > gpurun_out/${TAG}_gpu_tests.log 2>&1; echo "tests rc=$?"
tail -15 gpurun_out/${TAG}_gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/${TAG}_smoke.log
timeout 600 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/${TAG}_bench.log 2>&1; echo "bench rc=$?"
tail -1 gpurun_out/${TAG}_bench.log
