set -u
mkdir -p gpurun_out
T=r02i
timeout 300 python tools/prep_time.py > gpurun_out/${T}_prep.log 2>&1
FA3B_K5_PERSIST=1 timeout 300 python tools/prep_time.py >> gpurun_out/${T}_prep.log 2>&1; echo "prep rc=$?"
bash tools/ncu_prep.sh ${T}_k5_np
bash tools/ncu_prep.sh ${T}_k5_p FA3B_K5_PERSIST=1
bash tools/ncu_fwd.sh ${T}_prof_fp8_d128 128 0 1
