set -u
mkdir -p gpurun_out
T=r02by
bash tools/ncu_fwd.sh ${T}_prof_bf16_d256 256 0 0
