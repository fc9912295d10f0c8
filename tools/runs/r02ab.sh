set -u
mkdir -p gpurun_out
T=r02ab
bash tools/ncu_bwd.sh ${T}_prof_bwd_d128 128 0
bash tools/ncu_bwd.sh ${T}_prof_bwd_d64 64 0
