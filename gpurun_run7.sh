timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/gpu_tests.log 2>&1; echo tests=$?; tail -5 gpurun_out/gpu_tests.log
for s in 4 2 8; do
timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e --strip $s > gpurun_out/bench_s$s.log 2>&1; echo strip=$s rc=$?; tail -1 gpurun_out/bench_s$s.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['roofline']['ms_per_view'], d['roofline']['K_used'])"
done
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --init random > gpurun_out/bench_r.log 2>&1; echo random rc=$?; tail -1 gpurun_out/bench_r.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['roofline']['ms_per_view'])"
