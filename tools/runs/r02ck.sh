set -u
mkdir -p gpurun_out
T=r02ck
for i in 1 2 3; do timeout 1200 python -m pytest tests -q -m gpu -p no:randomly > gpurun_out/${T}_pytest_gpu_$i.log 2>&1; echo "pytest $i rc=$?"; done
