timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/gpu_tests.log 2>&1; echo tests=$?; grep -E "passed|failed|Error|assert " gpurun_out/gpu_tests.log | tail -12
