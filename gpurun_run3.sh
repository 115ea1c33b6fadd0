set -x
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/gpu_tests.log 2>&1; echo tests=$?; tail -15 gpurun_out/gpu_tests.log
timeout 600 python bench.py --steps 30 --warmup 3 --no-cpu-baseline > gpurun_out/bench_gt.log 2>&1; echo bench=$?; tail -2 gpurun_out/bench_gt.log
timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e --init random > gpurun_out/bench_rand.log 2>&1; echo bench=$?; tail -1 gpurun_out/bench_rand.log
timeout 300 python bench.py --profile-steps 2 --steps 2 --warmup 3 > gpurun_out/plain.log 2>&1 && timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/launches.csv python bench.py --profile-steps 2 --steps 2 --warmup 3 > gpurun_out/ncu1.log 2>&1; echo ncu1=$?
timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:raster -c 2 -o gpurun_out/prof_raster python bench.py --profile-steps 2 --steps 2 --warmup 3 > gpurun_out/ncu2.log 2>&1; echo ncu2=$?
