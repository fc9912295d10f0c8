#!/bin/bash
# One GPU session: tests, smoke, bench (both arms), ncu launch list + full capture.
# Usage (under gpurun): bash tools/gpu_round.sh <tag> [steps...]
set -u
TAG=${1:-r01}
shift || true
STEPS=${@:-"tests smoke bench ref ncu"}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/${TAG}_smi.txt 2>&1
for s in $STEPS; do
  case $s in
    tests) timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/${TAG}_pytest_gpu.log 2>&1; echo "pytest rc=$?" ;;
    smoke) timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo "smoke rc=$?" ;;
    bench) timeout 600 python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err; echo "bench rc=$?" ;;
    ref) timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/${TAG}_bench_ref.json 2> gpurun_out/${TAG}_bench_ref.err; echo "ref rc=$?" ;;
    ncu)
      timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv \
        --log-file gpurun_out/${TAG}_launches.csv python bench.py --steps 10 --warmup 3 --no-sweep --no-cpu-baseline > /dev/null 2>&1; echo "ncu-launches rc=$?"
      timeout 900 ncu --set full --clock-control none --import-source on -k regex:fa3b_fwd_kernel -s 3 -c 1 \
        -o gpurun_out/${TAG}_prof_fwd python bench.py --steps 5 --warmup 3 --no-sweep --no-cpu-baseline > gpurun_out/${TAG}_ncu_full.log 2>&1; echo "ncu-full rc=$?" ;;
  esac
done
