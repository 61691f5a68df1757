#!/bin/bash
# Whole-bench-step sweep of knob settings (B2K_TUNE), interleaved repeats on one box.
SETTINGS=("${@}")
if [ ${#SETTINGS[@]} -eq 0 ]; then SETTINGS=(""); fi
for r in 1 2 3; do
  for s in "${SETTINGS[@]}"; do
    B2K_TUNE="$s" python bench.py --no-cpu --no-e2e --steps 20 --warmup 5 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('[$s]', round(d['value']), round(d['kernels']['transpose']['GBps']), round(d['kernels']['reduce']['GBps']))"
  done
done
