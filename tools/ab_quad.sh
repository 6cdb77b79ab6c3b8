#!/bin/bash
# A/B of compute_Y_quad builds (2J > 8): quick_time per build dir, parity on the default build
OUT=gpurun_out/${AB_OUT:-ab}
mkdir -p $OUT
for b in "$@"; do
  echo "== $b"; python tools/quick_time.py --lib=paper_2011_12875_b200/$b/libsnapgpu.so 32,32,16,14 16,16,16,12 16,16,16,10 16,16,16,11 16,16,16,13
done > $OUT/ab.log 2>&1
cat $OUT/ab.log
