PRECS=tf32x3 timeout 300 python tools/fc1_trace.py 2>&1 | head -12
SIMNET_DIAG_FC1_A_EARLY=1 PRECS=tf32x3 timeout 300 python tools/fc1_trace.py 2>&1 | head -12
SIMNET_DIAG_FC1_SKIP_W=1 PRECS=tf32x3 timeout 300 python tools/fc1_trace.py 2>&1 | head -12
for v in X=0 SIMNET_DIAG_FC1_A_EARLY=1 SIMNET_DIAG_FC1_SKIP_W=1; do env $v timeout 120 python profiles/prof_run.py --precision tf32x3 --runs 2 | sed "s|^|[$v] |"; done
