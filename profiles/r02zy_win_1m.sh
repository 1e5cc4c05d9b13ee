# c5 at 1,048,576 sub-traces (96 rounds): overlapped-upload window size (SIMNET_WIN_ROUNDS) vs the default 16
for v in X=0 SIMNET_WIN_ROUNDS=48 SIMNET_WIN_ROUNDS=96 SIMNET_NO_UPLOAD_OVERLAP=1; do
  env $v N=100000000 K=1048576 timeout 900 python tools/e2e_c3.py 2>&1 | tail -2 | sed "s|^|[$v] |"
done
