#!/bin/bash
# ncu --set full of the 8-column persistent dense PCG with the Nystrom preconditioner (n = 1e5, ell = 2000):
# the third persistent launch of tools/mu_batch_timing.py is the first 8-column solve
ncu --set full --import-source on --clock-control none -k regex:pcg_persistent -s 2 -c 1 \
    -o gpurun_out/ncu_mu_batch_S8 -f python tools/mu_batch_timing.py > gpurun_out/ncu_mu_batch_S8.log 2>&1
echo ncu_rc=$?
