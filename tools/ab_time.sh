# A/B: quick_time of several builds (args: build dirs), then the parity tests on the default build
for b in "$@"; do
  echo "== $b"; python tools/quick_time.py --lib=paper_2011_12875_b200/$b/libsnapgpu.so 10,10,10,8 64,64,32,8
done > gpurun_out/ab.log 2>&1
python -m pytest tests/test_gpu_parity.py tests/test_gpu_determinism.py -x -q > gpurun_out/par.log 2>&1
