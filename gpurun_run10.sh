timeout 900 python -m pytest tests -m gpu -q > gpurun_out/gpu_tests.log 2>&1; echo tests=$?; grep -E "passed|failed|Error|assert " gpurun_out/gpu_tests.log | tail -12
timeout 900 python bench.py --config 4 --steps 20 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_c4.log 2>&1; echo c4=$?; tail -1 gpurun_out/bench_c4.log
timeout 600 python bench.py --config 2 --steps 20 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_c2.log 2>&1; echo c2=$?; tail -1 gpurun_out/bench_c2.log
timeout 300 python bench.py --config 1 --steps 50 --warmup 3 --no-e2e > gpurun_out/bench_c1.log 2>&1; echo c1=$?; tail -1 gpurun_out/bench_c1.log
