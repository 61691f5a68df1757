#!/bin/bash
# full GPU check with the cp.async default + ncu of the bench command
bash tools/r02_check.sh
bash tools/ncu_bench.sh
