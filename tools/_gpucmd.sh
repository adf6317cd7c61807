timeout 600 python -m pytest tests/test_gpu_fullsize.py -m gpu -x -q -k "walk_variants" > gpurun_out/gpu_tests.log 2>&1; tail -15 gpurun_out/gpu_tests.log
