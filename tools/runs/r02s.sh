set -u
mkdir -p gpurun_out
T=r02s
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/${T}_smi.txt 2>&1
timeout 600 python tools/ab.py paper_2407_08608_b200/libfa3b.so build/variants/psplit.so > gpurun_out/${T}_psplit_ab.log 2>&1; echo "ab rc=$?"
timeout 900 python bench.py > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err; echo "bench rc=$?"
timeout 300 python bench.py --dtype e4m3 --no-sweep --no-cpu-baseline > gpurun_out/${T}_bench_fp8.json 2> gpurun_out/${T}_bench_fp8.err; echo "fp8 rc=$?"
timeout 300 python bench.py --workload c5 --no-sweep --no-cpu-baseline > gpurun_out/${T}_bench_c5.json 2> gpurun_out/${T}_bench_c5.err; echo "c5 rc=$?"
timeout 300 python bench.py --workload c5 --dtype e4m3 --no-sweep --no-cpu-baseline > gpurun_out/${T}_bench_c5_fp8.json 2> gpurun_out/${T}_bench_c5_fp8.err; echo "c5fp8 rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/${T}_launches.csv python bench.py --steps 10 --warmup 3 --no-sweep --no-cpu-baseline > /dev/null 2>&1; echo "ncu-launches rc=$?"
bash tools/ncu_fwd.sh ${T}_prof_bf16_d128 128 0 0
bash tools/ncu_fwd.sh ${T}_prof_fp8_d128 128 0 1
bash tools/ncu_prep.sh ${T}_k5
