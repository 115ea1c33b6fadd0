timeout 900 python bench.py --steps 50 --warmup 5 > gpurun_out/bench_full.log 2>&1; echo bench=$?; tail -1 gpurun_out/bench_full.log
timeout 300 python bench.py --profile-steps 2 --steps 2 --warmup 3 > gpurun_out/plain.log 2>&1 && timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/launches.csv python bench.py --profile-steps 2 --steps 2 --warmup 3 > gpurun_out/ncu1.log 2>&1; echo ncu1=$?
timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:raster -c 2 -o gpurun_out/prof_raster python bench.py --profile-steps 1 --steps 2 --warmup 3 > gpurun_out/ncu2.log 2>&1; echo ncu2=$?
nproc; lscpu | grep "Model name"
