#!/bin/bash
# A/B every abtest/libb200k_*.so build on one box, twice, interleaved.
for r in 1 2; do for f in abtest/libb200k_*.so; do python tools/ab_lib.py $f; done; done
