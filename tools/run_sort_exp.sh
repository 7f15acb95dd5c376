#!/bin/bash
# sort micro-benchmark experiments on the GPU box (dev tool)
N=${SB_N:-7340032}
for cfg in "" "-DSORT_EXP=1" "-DSORT_EXP=2" "-DSORT_LB=32" "-DSORT_LB=8"; do
  SB_FLAGS="$cfg" ./tools/sortbench.sh > gpurun_out/sb_build.log 2>&1 || { cat gpurun_out/sb_build.log; exit 1; }
  for v in 1 0; do echo "== [$cfg] variant $v"; ./build/sortbench $N 24 stencil 10 $v | grep -E "median|verify"; done
  echo "== [$cfg] phases (persistent)"; ./build/sortbench_t $N 24 stencil 5 1 | grep phase
done
