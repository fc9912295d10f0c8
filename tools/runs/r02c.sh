set -u
mkdir -p gpurun_out
T=r02c
for i in 1 2; do
FA3B_FWD_WIDE=0 timeout 300 python tools/wide_ab.py >> gpurun_out/${T}_wide.log 2>&1
FA3B_FWD_WIDE=1 timeout 300 python tools/wide_ab.py >> gpurun_out/${T}_wide.log 2>&1
done
echo done
