timeout 900 python -m pytest tests -m gpu -q > gpurun_out/gpu_tests.log 2>&1; echo tests=$?; grep -E "passed|failed|Error|assert " gpurun_out/gpu_tests.log | tail -12
timeout 600 python bench.py --config 5 --steps 20 --warmup 3 > gpurun_out/bench_c5.log 2>&1; echo c5=$?; tail -2 gpurun_out/bench_c5.log
timeout 600 python bench.py --steps 30 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c3.log 2>&1; echo c3=$?; tail -1 gpurun_out/bench_c3.log
