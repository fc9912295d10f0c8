set -u
mkdir -p gpurun_out
T=r02b
./tools/ex2_bench > gpurun_out/${T}_ex2_bench.txt 2>&1
timeout 1500 python -m pytest tests -x -q -m gpu --durations=20 > gpurun_out/${T}_pytest_gpu.log 2>&1; echo "pytest rc=$?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err; echo "bench rc=$?"
timeout 300 python bench.py --workload c5 --no-cpu-baseline --steps 20 > gpurun_out/${T}_bench_c5.json 2> gpurun_out/${T}_bench_c5.err; echo "c5 rc=$?"
timeout 300 python bench.py --workload c5 --dtype e4m3 --no-cpu-baseline --steps 20 > gpurun_out/${T}_bench_c5_fp8.json 2> gpurun_out/${T}_bench_c5_fp8.err; echo "c5fp8 rc=$?"
timeout 300 python bench.py --dtype e4m3 --no-cpu-baseline --steps 20 > gpurun_out/${T}_bench_fp8.json 2> gpurun_out/${T}_bench_fp8.err; echo "fp8 rc=$?"
