set -u
mkdir -p gpurun_out
T=r02v
FA3B_FWD_Q1=1 timeout 600 python -m pytest tests/test_fwd_gpu.py tests/test_fp8_gpu.py -x -q -k "matches_oracle or error_band or full_size or many_items" > gpurun_out/${T}_pytest_q1.log 2>&1; echo "pytest q1 rc=$?"
FA3B_FWD_Q1=0 timeout 300 python tools/wide_ab.py > gpurun_out/${T}_q1_ab.log 2>&1
FA3B_FWD_Q1=1 timeout 300 python tools/wide_ab.py >> gpurun_out/${T}_q1_ab.log 2>&1
FA3B_FWD_Q1=0 timeout 300 python tools/wide_ab.py >> gpurun_out/${T}_q1_ab.log 2>&1
FA3B_FWD_Q1=1 timeout 300 python tools/wide_ab.py >> gpurun_out/${T}_q1_ab.log 2>&1; echo "ab rc=$?"
