set -u
mkdir -p gpurun_out
T=r02bv
for i in 1 2; do for TH in 4 5 6; do FA3B_FP8_THR=$TH timeout 600 python tools/wide_ab.py 2>/dev/null | grep e4m3 >> gpurun_out/${T}_thr_speed.log; done; done; echo "speed done"
for TH in 5; do FA3B_FP8_THR=$TH timeout 900 python tools/fp8_acc.py >> gpurun_out/${T}_thr_acc.log 2>&1; done; echo "acc done"
