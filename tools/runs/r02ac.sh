set -u
mkdir -p gpurun_out
T=r02ac
bash tools/ncu_c5.sh ${T}_prof_c5_bf16 0
bash tools/ncu_c5.sh ${T}_prof_c5_fp8 1
bash tools/ncu_fwd.sh ${T}_prof_fp8_d128 128 0 1
timeout 300 python bench.py --dtype e4m3 --no-sweep --no-cpu-baseline > gpurun_out/${T}_bench_fp8.json 2> gpurun_out/${T}_bench_fp8.err; echo "fp8 rc=$?"
timeout 300 python bench.py --workload c5 --dtype e4m3 --no-sweep --no-cpu-baseline > gpurun_out/${T}_bench_c5_fp8.json 2> gpurun_out/${T}_bench_c5_fp8.err; echo "c5fp8 rc=$?"
