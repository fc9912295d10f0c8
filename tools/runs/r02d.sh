set -u
mkdir -p gpurun_out
T=r02d
timeout 900 python -m pytest tests/test_fp8_gpu.py -x -q > gpurun_out/${T}_fp8_tests.log 2>&1; echo "fp8 tests rc=$?"
for thr in 0 1 2; do
FA3B_FP8_THR=$thr FA3B_FWD_WIDE=0 timeout 300 python tools/wide_ab.py >> gpurun_out/${T}_thr.log 2>&1
done
timeout 300 python tools/wide_ab.py >> gpurun_out/${T}_thr.log 2>&1
echo done
