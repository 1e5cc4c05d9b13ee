# diagnostics: per-round time with parts of the fused round knocked out (results invalid by design)
for KO in 0 1 2 4 8 12; do SIMNET_KNOCKOUT=$KO timeout 120 python profiles/prof_run.py --precision tf32x3 --runs 2 | sed "s/^/KO=$KO /"; done
for KO in 0 4 8; do SIMNET_KNOCKOUT=$KO timeout 120 python profiles/prof_run.py --precision bf16 --runs 2 | sed "s/^/KO=$KO /"; done
