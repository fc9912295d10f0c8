set -u
mkdir -p gpurun_out
T=r02e
bash tools/gpu_round.sh $T tests smoke bench ncu
bash tools/ncu_fwd.sh ${T}_prof_fp8_d128 128 0 1
