timeout 1800 python -m pytest tests/test_gpu_fullsize.py -x -q 2>&1 | tail -25 > gpurun_out/r2ft.log
cat gpurun_out/r2ft.log
