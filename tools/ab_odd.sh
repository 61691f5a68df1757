#!/bin/bash
# interleaved A/B of abl/libA.so vs abl/libB.so (+ optional knob sets) on odd shapes
for r in 1 2; do
  for L in A B; do B2K_LIB=$PWD/abl/lib$L.so python tools/ab_odd.py; done
  for T in "transpose.scalar_ctas=2" "transpose.scalar_ctas=3" "transpose.scalar_ctas=4"; do
    B2K_LIB=$PWD/abl/libB.so B2K_TUNE=$T python tools/ab_odd.py; done
done
