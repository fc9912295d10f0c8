set -u
mkdir -p gpurun_out
T=r02o
timeout 900 python -m pytest tests/test_bwd_gpu.py -x -q > gpurun_out/${T}_pytest_bwd.log 2>&1; echo "pytest bwd rc=$?"
timeout 1500 compute-sanitizer --tool racecheck --print-limit 50 python tools/sanitize_cases.py > gpurun_out/${T}_sanitize_racecheck.log 2>&1; echo "racecheck rc=$?"
