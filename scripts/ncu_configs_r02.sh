#!/bin/bash
# ncu --set full of the sweep kernels of configs 3 and 4 (vertex-owned engine, host loop so that ncu sees the kernels)
for c in c3 c4; do
  HLM_B200_CREW_HOST_LOOP=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_c2_argmax_light|k_c2_argmax_task|k_c2_check|k_c2_kill_light" -c 12 \
    -o gpurun_out/crew_${c}_r02 python scripts/crew_ncu_target.py $c 2>&1 | tail -2
done
