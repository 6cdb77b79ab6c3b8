for b in _build _build_nl8 _build_nl12; do
ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none -k regex:k_nl_lists -s 2 -c 6 --csv python tools/pos_probe.py --lib=paper_2011_12875_b200/$b/libsnapgpu.so 8 2>/dev/null > gpurun_out/pos_warm_$b.csv
done
