bash tools/ab_time.sh _build_head _build
python tools/e2e_parts.py > gpurun_out/e2e_parts22.log 2>&1
python -m pytest tests/test_gpu_determinism.py tests/test_gpu_parity.py -q -x > gpurun_out/par2.log 2>&1
