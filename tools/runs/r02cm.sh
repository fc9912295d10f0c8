set -u
mkdir -p gpurun_out
T=r02cm
FA3B_FWD_WIDE256=1 timeout 900 python -m pytest tests/test_fwd_gpu.py tests/test_fp8_gpu.py -x -q -k "256 or d256 or matches_oracle or error_band or tiny" > gpurun_out/${T}_pytest_wide256.log 2>&1; echo "pytest rc=$?"
for i in 1 2; do for W in 0 1; do AB_DIMS=256 FA3B_FWD_WIDE256=$W timeout 600 python tools/wide_ab.py 2>/dev/null >> gpurun_out/${T}_wide256.log; done; done; echo "speed done"
