set -u
mkdir -p gpurun_out
T=r02bi
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${T}_launches.csv python bench.py --steps 3 --warmup 3 --no-sweep --no-cpu-baseline > gpurun_out/${T}_ncu_bench.log 2>&1; echo "ncu launches rc=$?"
bash tools/ncu_fwd.sh ${T}_prof_bf16_d128 128 0 0
bash tools/ncu_fwd.sh ${T}_prof_fp8_d128 128 0 1
