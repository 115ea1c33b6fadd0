for s in 8 4 2; do
timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e --strip $s > gpurun_out/bench_s$s.log 2>&1; echo strip=$s rc=$?; tail -1 gpurun_out/bench_s$s.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['roofline']['ms_per_view'])"
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --strip $s --init random > gpurun_out/bench_r$s.log 2>&1; echo strip=$s random rc=$?; tail -1 gpurun_out/bench_r$s.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['roofline']['ms_per_view'])"
done
