# per-kernel device durations (ncu, serialised) of one force step: kdur.sh BUILD NX NY NZ
ncu --metrics gpu__time_duration.sum,smsp__warp_issue_stalled_no_instruction_per_warp_active.pct --clock-control none -s 8 -c 8 --csv \
  python tools/quick_time.py --lib=paper_2011_12875_b200/$1/libsnapgpu.so $2,$3,$4,8 2>/dev/null | grep -E "k_compute|k_y_finish|k_fused|k_gather" | awk -F'","' '{print $5, $(NF-2), $NF}'
