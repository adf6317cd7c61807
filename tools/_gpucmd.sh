bash tools/_ab.sh
SVR_LIB_PATH=$PWD/abtmp/shape2.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -m gpu -x -q > gpurun_out/gpu_tests_s2.log 2>&1; tail -3 gpurun_out/gpu_tests_s2.log
