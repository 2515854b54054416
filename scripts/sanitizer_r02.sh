#!/bin/bash
# compute-sanitizer passes over the round-2 kernels -> profiles/sanitizer_r02.txt (run on the GPU box)
out=gpurun_out/sanitizer_r02.txt
: > $out
run() { echo "== $*" >> $out; timeout 900 "$@" 2>&1 | grep -E "passed|failed|ERROR SUMMARY|RACECHECK SUMMARY|same|DIFFERENT|ok=|Error|error" | tail -12 >> $out; }
K="test_gpu_multi or test_gpu_variants or test_gpu_fused or edge_case or loader or test_crew"
run compute-sanitizer --tool memcheck python -m pytest tests -m gpu -q -k "$K"
run compute-sanitizer --tool initcheck python -m pytest tests -m gpu -q -k "$K"
HLM_B200_CREW_HOST_LOOP=1 FIRST_VARIANT=crew run compute-sanitizer --tool racecheck python scripts/crew_small.py
FIRST_VARIANT=crew run compute-sanitizer --tool memcheck python scripts/crew_small.py
run compute-sanitizer --tool memcheck python scripts/shard_check.py uniform 20000 30000 4 1,3
# racecheck follows neither conditional graph nodes nor NCCL's kernels: host-driven loops, co-located exchange
HLM_B200_CREW_HOST_LOOP=1 run compute-sanitizer --tool racecheck python scripts/shard_check.py powerlaw 20000 40000 0 2 nonccl
# the one-launch kernel of small instances (cooperative grid, shared-memory scans, grid barriers)
run compute-sanitizer --tool racecheck python -m pytest tests/test_gpu_fused.py -m gpu -q
run compute-sanitizer --tool synccheck python -m pytest tests/test_gpu_fused.py -m gpu -q
cat $out
