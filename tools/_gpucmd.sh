timeout 900 python -m pytest tests -m gpu -x -q -k "tri or cfg5" > gpurun_out/gpu_tests.log 2>&1; tail -3 gpurun_out/gpu_tests.log
bash tools/_ab_cfg.sh cfg5
