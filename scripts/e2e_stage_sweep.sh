#!/bin/bash
# pageable e2e of config 2 over staging-ring shapes
lscpu | grep -E "Model name|L3|L2|Socket|NUMA node\(s\)" 
for cfg in "8192 24" "2048 24" "2048 8" "1024 32" "512 32" "4096 8" "4096 48"; do
  set -- $cfg
  echo "chunk_kb=$1 slots=$2"
  HLM_B200_STAGE_CHUNK_KB=$1 HLM_B200_STAGE_SLOTS=$2 python scripts/e2e_pageable.py 2>&1 | tail -1
done
