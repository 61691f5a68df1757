#!/bin/bash
# Run-to-run spread of the bench line on one box (N runs of the default bench).
N=${1:-8}
for i in $(seq 1 $N); do
  python bench.py --no-cpu 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(json.dumps({'value': d['value'], 'transpose': d['kernels']['transpose']['GBps'], 'reduce': d['kernels']['reduce']['GBps'], 'e2e': d['e2e']['value'], 'sm_mhz': d['clocks']['sm_mhz'], 'reasons': d['clocks']['reasons']}))"
done
