set -u
mkdir -p gpurun_out
T=r02af
for rep in 1 2; do
  for e in warp cta; do
    echo "== FA3B_FWD_PAIRING=$e" >> gpurun_out/${T}_pairing_short.log
    FA3B_FWD_PAIRING=$e timeout 300 python tools/short_ab.py paper_2407_08608_b200/libfa3b.so >> gpurun_out/${T}_pairing_short.log 2>&1
  done
done
echo done
