#!/bin/bash
# ncu --set full of k_rounds_fused on config 1 (one launch = the whole matching): after the probe's warm-up calls
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_rounds_fused" -s 3 -c 1 -f \
  -o gpurun_out/fused_c1_r02 python scripts/fused_trace.py c1only 2>&1 | tail -3
