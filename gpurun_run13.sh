timeout 900 python -m pytest tests -m gpu -q > gpurun_out/gpu_tests.log 2>&1; echo tests=$?; grep -E "passed|failed|Error|assert " gpurun_out/gpu_tests.log | tail -12
for s in 4 2 8; do
timeout 300 python bench.py --steps 30 --warmup 3 --no-cpu-baseline --no-e2e --strip $s > gpurun_out/bench_s$s.log 2>&1; echo strip=$s rc=$?; tail -1 gpurun_out/bench_s$s.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['roofline']['ms_per_view'], d['roofline']['K_used'])"
done
