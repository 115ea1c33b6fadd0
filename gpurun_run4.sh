timeout 900 python -m pytest tests -m gpu -q > gpurun_out/gpu_tests.log 2>&1; echo tests=$?; tail -5 gpurun_out/gpu_tests.log
timeout 600 python bench.py --steps 30 --warmup 3 --no-cpu-baseline > gpurun_out/bench_gt.log 2>&1; echo bench=$?; tail -1 gpurun_out/bench_gt.log
timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e --init random > gpurun_out/bench_rand.log 2>&1; echo bench=$?; tail -1 gpurun_out/bench_rand.log
