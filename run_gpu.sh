timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?; tail -15 gpurun_out/pytest_gpu.log
timeout 300 python bench.py --algo dense --n 20000 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:solve_kernel -s 2 -c 1 -o gpurun_out/r01_prof_dense python bench.py --algo dense --n 20000 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ncu2.log 2>&1; echo ncu rc=$?
