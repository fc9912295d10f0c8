set -u
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/r02a_smi.txt 2>&1
nproc > gpurun_out/r02a_nproc.txt
./tools/ex2_bench > gpurun_out/r02a_ex2_bench.txt 2>&1
timeout 1500 python -m pytest tests -x -q -m gpu --durations=15 > gpurun_out/r02a_pytest_gpu.log 2>&1; echo "pytest rc=$?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02a_smoke.log 2>&1; echo "smoke rc=$?"
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/r02a_bench.json 2> gpurun_out/r02a_bench.err; echo "bench rc=$?"
