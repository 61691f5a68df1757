#!/bin/bash
# A/B the bench step between abtest/libb200k_*.so builds on one box (interleaved).
for r in 1 2 3; do
  for f in abtest/libb200k_*.so; do
    B2K_LIB=$PWD/$f python bench.py --no-cpu --no-e2e --steps 20 --warmup 5 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$f', round(d['value']), round(d['kernels']['transpose']['GBps']), round(d['kernels']['reduce']['GBps']))"
  done
done
