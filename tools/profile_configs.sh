#!/bin/bash
# ncu captures of U / Y / dE / gather at the BASELINE.json configs (run under gpurun):
#   bash tools/profile_configs.sh OUTDIR
# One launch of each kernel after a warm-up step (direct launches: stage
# timing on), --set full plus the thread-level FP64 op counters.
OUT=${1:-gpurun_out/prof}
mkdir -p $OUT
M=sm__sass_thread_inst_executed_op_dfma_pred_on.sum,sm__sass_thread_inst_executed_op_dmul_pred_on.sum,sm__sass_thread_inst_executed_op_dadd_pred_on.sum
for cfg in "C2 10 10 10 8" "C3 64 64 32 8" "C4 32 32 16 14"; do
  set -- $cfg
  ncu --set full --metrics $M --clock-control none --import-source on \
      -k regex:'k_compute_U|k_compute_Y|k_fused_dE|k_gather' -s 4 -c 4 \
      -o $OUT/$1 python tools/profile_step.py $2 $3 $4 $5 2 > $OUT/$1.log 2>&1
done
# launch list of the bench command (per-kernel shares of the step)
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file $OUT/launches_C2.csv python bench.py --steps 20 --warmup 3 --no-e2e \
    --no-cpu-baseline --no-probe > $OUT/launches_C2.log 2>&1
