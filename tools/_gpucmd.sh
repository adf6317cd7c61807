timeout 900 python -m pytest tests -m gpu -x -q -k "fan or cfg3 or fullsize or parity" > gpurun_out/gpu_tests.log 2>&1; tail -2 gpurun_out/gpu_tests.log
bash tools/_ab_cfg.sh cfg3
