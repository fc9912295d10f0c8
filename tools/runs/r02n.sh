set -u
mkdir -p gpurun_out
T=r02n
bash tools/ncu_fwd.sh ${T}_prof_fp8_d128 128 0 1
bash tools/ncu_fwd.sh ${T}_prof_bf16_d128 128 0 0
bash tools/sanitize.sh ${T}
