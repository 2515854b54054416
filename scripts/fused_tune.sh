#!/bin/bash
# k_rounds_fused: sweep form (plain / pipelined) x CTAs per SM on small uniform instances
for pipe in 0 1; do for ctas in 1 2 3 4; do
  echo "== pipe $pipe ctas $ctas"
  HLM_B200_FUSED_PIPE=$pipe HLM_B200_FUSED_CTAS=$ctas timeout 200 python scripts/fused_probe.py fusedonly
done; done
