set -u
mkdir -p gpurun_out
T=r02y
for thr in 2 3 4 6; do
  FA3B_FP8_THR=$thr timeout 300 python tools/wide_ab.py 2>&1 | grep e4m3 | grep '"d": 128' >> gpurun_out/${T}_thr_ab.log
  FA3B_FP8_THR=$thr timeout 300 python tools/fp8_acc.py >> gpurun_out/${T}_thr_acc.log 2>&1
done
echo done
