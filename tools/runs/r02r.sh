set -u
mkdir -p gpurun_out
T=r02r
timeout 1500 python -m pytest tests -x -q -m gpu --durations=15 > gpurun_out/${T}_pytest_gpu.log 2>&1; echo "pytest rc=$?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.log 2>&1; echo "smoke rc=$?"
