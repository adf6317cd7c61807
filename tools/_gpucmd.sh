SVR_LIB_PATH=$PWD/abtmp/ty4.so timeout 900 python -m pytest tests -m gpu -x -q -k "fill or fullsize" > gpurun_out/gpu_tests.log 2>&1; tail -2 gpurun_out/gpu_tests.log
bash tools/_ab.sh
