timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?; tail -2 gpurun_out/pytest_gpu.log
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo smoke rc=$?
timeout 900 python bench.py > gpurun_out/bench_r01.json 2> gpurun_out/bench_r01.err; echo bench rc=$?; cat gpurun_out/bench_r01.json
timeout 900 python bench.py --precision fp32 --no-cpu-baseline > gpurun_out/bench_r01_fp32.json 2>/dev/null; cat gpurun_out/bench_r01_fp32.json | cut -c1-200
timeout 900 python bench.py --algo dense --n 50000 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_r01_dense.json 2>/dev/null; cat gpurun_out/bench_r01_dense.json | cut -c1-200
timeout 300 python bench.py --n 100000 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r01_launches.csv python bench.py --n 100000 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ncu1.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:solve_kernel -s 2 -c 1 -o gpurun_out/r01_prof_env python bench.py --n 100000 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ncu2.log 2>&1; echo ncu rc=$?
